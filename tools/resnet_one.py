import sys
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn
from paper_1903_01855_b200.workloads import resnet
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=32, mode=sys.argv[1] if len(sys.argv) > 1 else "staged", image=224, seed=0)
for _ in range(3): tr.step()
_native.sync(0)
