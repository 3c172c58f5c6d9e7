"""Dev tool (CPU): trace a workload, lower it, dump/compile its fused kernels.

Constant folding needs the GPU; this tool substitutes a numpy evaluator for
the handful of folded ops so codegen can be iterated on a GPU-less host.
Never used by the product or the tests.
"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import executor, lowering, rowfuse, _native, plugins
from paper_1903_01855_b200.tensor import Tensor

def np_fold(node, inputs, library):
    from oracle import kernels_np as K
    arrs = [t.raw() for t in inputs]
    op, at = node.op, node.attrs
    if op == "reshape": out = arrs[0].reshape(at["shape"])
    elif op == "broadcast_to": out = np.broadcast_to(arrs[0], at["shape"]).copy()
    elif op == "constant": return [at["value"]]
    elif op in ("reduce_sum", "reduce_mean"): out = getattr(K, op)(arrs[0], at.get("axes"), at.get("keepdims", False))
    elif op == "transpose": out = arrs[0].T.copy()
    else: out = K.KERNELS[op](*arrs)
    out = np.asarray(out); out.flags.writeable = False
    return [Tensor._adopt(inputs[0].dtype if op != "greater" else sf.boolean, out.shape, inputs[0].device, None, out)]

executor.run_node_for_folding = np_fold
import paper_1903_01855_b200.graph as g
g.constant_fold.__globals__["run_node_for_folding"] = np_fold

from paper_1903_01855_b200.workloads import l2hmc
import os
l2hmc.N_STEPS = int(os.environ.get("NSTEPS", "10"))
plugins.install()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 200
s = l2hmc.L2HMCSampler(sf, B, "staged", seed=0)
pf = s.transition
bound = pf._bind((s.x,), {})
cf = pf._trace_to_concrete(bound)
gf = cf.graph
print("nodes", len(gf.nodes), gf.op_counts())
lw = lowering.Lowerer(0, "device")
ins = []
for ph in gf.inputs:
    ins.append(lw.new(ph.dtype, ph.shape, "input"))
outs = lw.lower_graph(gf, ins, ())
units = lowering.fuse(rowfuse.plan_rows(lw.ops), True)
print("units", [type(u).__name__ for u in units][:10], len(units))
import threading
from concurrent.futures import ThreadPoolExecutor
jobs=[]
for idx,u in enumerate(units):
    if isinstance(u, tuple):
        needed = {id(o) for o in outs}
        for later in units[idx+1:]:
            ops_ = later[0].ops if isinstance(later, tuple) else getattr(later, "ops", [later])
            for op in ops_:
                for x in op.ins: needed.add(id(x.root()))
        name, src = rowfuse.generate_rowprog(u[0], u[1], needed)[:2]
        jobs.append((name, src))
print("chunks", len(jobs), "max bytes", max(len(s) for _, s in jobs))
t=time.time()
if os.environ.get("COMPILE", "1") == "1":
    with ThreadPoolExecutor(8) as pool: list(pool.map(lambda j: _native.jit_compile(*j), jobs))
print("parallel compile", time.time()-t)
for i, (name, src) in enumerate(jobs):
    open(f"/tmp/chunk{i}.cu", "w").write(src)
