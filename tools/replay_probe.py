"""Dev probe (GPU): where time goes with whole-program graph replay (ResNet b32)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn, executor
from paper_1903_01855_b200.workloads import resnet
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=32, mode="staged", image=224, seed=0)
stats = {"try": 0, "hit": 0, "capture": 0}
orig_try = executor._ProgramGraph.try_run
def try_run(self, inputs):
    stats["try"] += 1
    r = orig_try(self, inputs)
    stats["hit"] += r is not None
    return r
executor._ProgramGraph.try_run = try_run
orig_init = executor._ProgramGraph.__init__
def init(self, *a, **k):
    stats["capture"] += 1
    t = time.perf_counter(); orig_init(self, *a, **k); print("capture", time.perf_counter() - t)
executor._ProgramGraph.__init__ = init
for i in range(6):
    t = time.perf_counter(); tr.step(); _native.sync(0); print("step", i, time.perf_counter() - t, dict(stats))
pr = cProfile.Profile(); pr.enable()
for _ in range(3): tr.step()
_native.sync(0); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(20)
