"""Dev probe (GPU): one steady-state staged ResNet-50 b32 step inside an NVTX
range "prof", for `ncu --nvtx --nvtx-include prof/` (per-kernel time of one step)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn
from paper_1903_01855_b200.workloads import resnet
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=int(sys.argv[1]) if len(sys.argv) > 1 else 32, mode="staged",
                        image=224, seed=0)
for _ in range(4):
    tr.step()
_native.sync(0)
torch.cuda.nvtx.range_push("prof")
tr.step()
_native.sync(0)
torch.cuda.nvtx.range_pop()
