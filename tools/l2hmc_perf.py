"""Dev probe: staged L2HMC step time at several chain counts (GPU)."""
import os, sys, time
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, plugins
from paper_1903_01855_b200.workloads import l2hmc

sf.init_runtime(sf.RuntimeOptions())
plugins.install()
for b in [int(x) for x in sys.argv[1:]] or [200, 100000]:
    s = l2hmc.L2HMCSampler(sf, b, "staged", seed=0)
    t0 = time.perf_counter(); s.step(); _native.sync(0); tc = time.perf_counter() - t0
    prog = next(iter(s.transition.cached_functions()[0].graph._plan.values()))
    seg = prog.segments[0]
    for _ in range(3): s.step()
    _native.sync(0)
    n = 20
    t = time.perf_counter()
    for _ in range(n): s.step()
    _native.sync(0)
    wall = (time.perf_counter() - t) / n
    seg.plan.profile(True)
    for _ in range(5): s.step()
    st = seg.plan.step_stats(); seg.plan.profile(False)
    kms = sum(ms / r for k, ms, r in st if r)
    print(f"chunk={os.environ.get('SF_CHUNK_COST','2500')} B={b}: compile {tc:.1f}s launches {prog.n_launches} "
          f"wall {wall*1e3:.3f} ms/step gpu {kms:.3f} ms -> {b/wall:.3e} samples/s", flush=True)
    if os.environ.get("SHOW_STEPS"):
        print("  per-step ms:", " ".join(f"{ms / r:.3f}" for k, ms, r in st if r))
