"""Generate (without a GPU) the row-program sources of a staged workload and
compile them with nvcc for SASS inspection.

    python tools/dump_rows.py OUTDIR [batch] [--inputs]

Traces the L2HMC transition on the host, runs the staged compiler's
lowering (Lowerer -> cse -> plan_rows -> generate_rowprog) and writes one
.cu per generated kernel plus sf_ops.cuh, then `nvcc -cubin` for sm_100a.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1903_01855_b200 as sf  # noqa: E402
from paper_1903_01855_b200 import plugins, rowfuse  # noqa: E402
from paper_1903_01855_b200.lowering import Lowerer, cse  # noqa: E402
from paper_1903_01855_b200.workloads import l2hmc  # noqa: E402


def _host_fold(node, inputs, library):
    """Dev-tool stand-in for constant folding without a GPU (numpy)."""
    import numpy as np

    from paper_1903_01855_b200.tensor import Tensor

    a = [x.raw() for x in inputs]
    op, at = node.op, node.attrs
    fns = {"mul": np.multiply, "add": np.add, "sub": np.subtract, "div": np.divide}
    if op in fns:
        r = fns[op](a[0], a[1])
    elif op == "neg":
        r = -a[0]
    elif op == "exp":
        r = np.exp(a[0])
    elif op == "reshape":
        r = a[0].reshape(at["shape"])
    elif op == "broadcast_to":
        r = np.broadcast_to(a[0], at["shape"])
    elif op == "transpose":
        r = a[0].T
    elif op == "matmul":
        r = a[0] @ a[1]
    elif op == "identity":
        r = a[0]
    elif op in ("reduce_sum", "reduce_mean"):
        f = np.sum if op == "reduce_sum" else np.mean
        r = f(a[0], axis=at.get("axes"), keepdims=at.get("keepdims", False))
    else:
        raise NotImplementedError(op)
    r = np.ascontiguousarray(r, dtype=inputs[0].dtype.np_dtype)
    r.flags.writeable = False
    return [Tensor(inputs[0].dtype, r.shape, inputs[0].device, array=r)]


def main():
    from paper_1903_01855_b200 import executor

    executor.run_node_for_folding = _host_fold
    out = sys.argv[1]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 100000
    draws = "inputs" if "--inputs" in sys.argv else "runtime"
    os.makedirs(out, exist_ok=True)
    sf.init_runtime(sf.RuntimeOptions())
    plugins.install()
    if "--c2" in sys.argv:
        from paper_1903_01855_b200.workloads import microbench

        ch = microbench.Chain("staged")
        pf = ch.fn
        args = [ch.x]
    elif "--leapfrog" in sys.argv:
        from paper_1903_01855_b200.workloads.leapfrog import Leapfrog

        wl = Leapfrog(batch, "staged")
        pf = wl.staged_functions[0]
        args = [wl.q, wl.p]
    else:
        s = l2hmc.L2HMCSampler(sf, batch, "staged", seed=0, draws=draws)
        args = [s.x] if draws == "runtime" else [s.x] + [
            sf.tensor_from_host(d.reshape(-1), d.shape, sf.float32) for d in s.host_draws()]
        pf = s.transition
    cf = pf._concrete_for(pf._bind(tuple(args), {}))
    gf = cf.graph
    lw = Lowerer(0, "device")
    lw.fold_captures = executor.BAKE  # as Program does
    ins = []
    values = list(args) + cf.materialize_captured()
    for i, (ph, v) in enumerate(zip(gf.inputs, values)):
        lv = lw.new(ph.dtype, ph.shape, "var" if ph.is_variable_ref else "input")
        lv.index = i
        if executor.bakeable(ph, v):  # as Program does
            lv.vals = v.raw().reshape(-1)
            lv.tensor = v
        ins.append(lv)
    outs = lw.lower_graph(gf, ins, ())
    keep = frozenset(id(v.root()) for v in outs)
    ops = cse(lw.ops)
    if executor.ELIDE_ZERO_ADDS:
        from paper_1903_01855_b200.lowering import elide_zero_adds
        ops = elide_zero_adds(ops, keep)
    units = rowfuse.plan_rows(ops, keep)
    k = 0
    shutil.copy(os.path.join(ROOT, "paper_1903_01855_b200", "csrc", "sf_ops.cuh"), out)
    for u, unit in enumerate(units):
        if isinstance(unit, tuple):
            # values read after this unit: later units' inputs and the outputs
            later = {id(x.root()) for v in units[u + 1:]
                     for op in (v[0].ops if isinstance(v, tuple) else [v])
                     for x in getattr(op, "ins", [])}
            needed = {id(o) for op in unit[0].ops for o in op.outs
                      if id(o) in keep or id(o) in later}
            name, src = rowfuse.generate_rowprog(unit[0], unit[1], needed)[:2]
            path = os.path.join(out, f"k{k}_{name}.cu")
            with open(path, "w") as f:
                f.write(src)
            r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin",
                                "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
                                "-Xptxas", "-v", "-I", out, "-o", path[:-3] + ".cubin", path],
                               capture_output=True, text=True)
            print(name, len(src.splitlines()), "lines", r.stderr.strip().splitlines()[-1:])
            k += 1


if __name__ == "__main__":
    main()
