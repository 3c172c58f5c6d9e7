"""Dev probe (GPU): which elementwise ops stay single-op launches in the staged ResNet step."""
import collections, sys
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn, executor
from paper_1903_01855_b200.workloads import resnet
seen = collections.Counter()
orig = executor.Program._emit_single_ew
def spy(self, pw, op, use, define):
    seen[(op.name, tuple(tuple(x.shape) for x in op.ins), tuple(op.outs[0].shape))] += 1
    return orig(self, pw, op, use, define)
executor.Program._emit_single_ew = spy
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=32, mode="staged", image=224, seed=0)
tr.step(); _native.sync(0)
for k, v in seen.most_common(40):
    print(v, k)
print("total", sum(seen.values()))
