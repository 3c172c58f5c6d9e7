"""Dev probe (GPU): host-side profile of the staged ResNet-50 b32 train step."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn
from paper_1903_01855_b200.workloads import resnet
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=32, mode="staged", image=224, seed=0)
for _ in range(3): tr.step()
_native.sync(0)
t = time.perf_counter()
for _ in range(5): tr.step()
host = (time.perf_counter() - t) / 5
_native.sync(0)
wall = (time.perf_counter() - t) / 5
print(f"host {host*1e3:.1f} ms/step, wall {wall*1e3:.1f} ms/step")
pr = cProfile.Profile(); pr.enable()
for _ in range(3): tr.step()
_native.sync(0)
pr.disable()
pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(35)
