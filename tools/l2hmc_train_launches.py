import sys, time; sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc
sf.init_runtime(sf.RuntimeOptions(seed=1)); plugins.install()
tr = l2hmc.L2HMCTrain(sf, 200, "staged", seed=0)
for _ in range(3): tr.step()
_native.sync(0)
l0 = _native.launch_count(0); t = time.perf_counter()
with sf.Tape() as tp:
    loss, x_out = tr.forward_loss(tr.x)
_native.sync(0); t1 = time.perf_counter(); l1 = _native.launch_count(0)
grads = tp.gradient(loss, tr.params)
_native.sync(0); t2 = time.perf_counter(); l2 = _native.launch_count(0)
tr.apply_updates(*grads)
_native.sync(0); t3 = time.perf_counter(); l3 = _native.launch_count(0)
print("fwd", l1-l0, (t1-t)*1e3, "bwd", l2-l1, (t2-t1)*1e3, "apply", l3-l2, (t3-t2)*1e3)
for pf in tr.staged_functions:
    for cf in pf.cached_functions():
        g = cf.graph
        print(pf._name, len(g.nodes), [ (p.n_launches, len(p.segments)) for p in (g._plan or {}).values()])
        fb = g._fwd_bwd
        if fb:
            fwd, bwd = fb[0], fb[1]
            print(" fwd variant", len(fwd.nodes), [(p.n_launches, len(p.segments)) for p in (fwd._plan or {}).values()])
            print(" bwd", len(bwd.graph.nodes), [(p.n_launches, len(p.segments)) for p in (bwd.graph._plan or {}).values()])
            for c in bwd.__dict__.get("_selected", {}).values():
                print(" bwd sel", len(c.graph.nodes), [(p.n_launches, len(p.segments)) for p in (c.graph._plan or {}).values()])
