"""Dev probe: ResNet-50 train step time (GPU)."""
import sys, time
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn
from paper_1903_01855_b200.workloads import resnet

b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for mode in sys.argv[2:] or ["staged", "eager"]:
    sf.init_runtime(sf.RuntimeOptions()); nn.install()
    tr = resnet.ResNetTrain(sf, batch=b, mode=mode, image=224, seed=0)
    t0 = time.perf_counter(); tr.step(); _native.sync(0); first = time.perf_counter() - t0
    tr.step(); _native.sync(0)
    n = 3
    t = time.perf_counter()
    for _ in range(n): tr.step()
    _native.sync(0)
    dt = (time.perf_counter() - t) / n
    print(f"resnet50 b={b} {mode}: first {first:.1f}s, {dt*1e3:.1f} ms/step, {b/dt:.1f} img/s, "
          f"{0.785e12*b/32/dt/1e12:.2f} TFLOP/s", flush=True)
