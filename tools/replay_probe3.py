"""Dev probe (GPU): who keeps the forward replay's outputs alive."""
import gc, sys
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn, executor
from paper_1903_01855_b200.tensor import Tensor
from paper_1903_01855_b200.workloads import resnet
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=8, mode="staged", image=64, seed=0)
for i in range(2):
    tr.step(); _native.sync(0)
# find live tensors backed by _GraphBuffer
live = [o for o in gc.get_objects() if isinstance(o, Tensor) and isinstance(o._buf, executor._GraphBuffer)]
print("live graph-backed tensors:", len(live))
def chain(o, depth=0, seen=None):
    seen = seen or set()
    if depth > 6: return
    for r in gc.get_referrers(o):
        if id(r) in seen or r is live or type(r).__name__ in ("frame", "function"): continue
        seen.add(id(r))
        desc = type(r).__name__
        if isinstance(r, dict): desc += str(list(r.keys())[:4])
        print("  " * depth, desc)
        if depth < 5: chain(r, depth + 1, seen)
if live:
    chain(live[0])
gc.collect()
live = [o for o in gc.get_objects() if isinstance(o, Tensor) and isinstance(o._buf, executor._GraphBuffer)]
print("after gc.collect:", len(live))
