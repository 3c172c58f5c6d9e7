"""Dev probe (GPU): why graph replays are refused."""
import gc, sys
sys.path.insert(0, ".")
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native, nn, executor
from paper_1903_01855_b200.state import Variable
from paper_1903_01855_b200.workloads import resnet
sf.init_runtime(sf.RuntimeOptions()); nn.install()
tr = resnet.ResNetTrain(sf, batch=8, mode="staged", image=64, seed=0)
orig_try = executor._ProgramGraph.try_run
def try_run(self, inputs):
    busy = self.token_ref is not None and self.token_ref() is not None
    mism = []
    for i, (k, v) in enumerate(zip(self.kinds, inputs)):
        if k[0] == "borrow":
            p = v._storage_ptr() if isinstance(v, Variable) else (v._buf.ptr if isinstance(v._buf, executor._GraphBuffer) else None)
            if p != k[1]: mism.append((i, type(v).__name__, type(v._buf).__name__ if hasattr(v, "_buf") else None))
    r = orig_try(self, inputs)
    print(f"  prog {self.prog.gf.name[:30]} busy={busy} mismatches={mism[:3]} n_in={len(inputs)} hit={r is not None}")
    if busy:
        t = self.token_ref()
        print("   referrers of token:", [type(x).__name__ for x in gc.get_referrers(t)][:5])
    return r
executor._ProgramGraph.try_run = try_run
for i in range(4):
    tr.step(); _native.sync(0); print("step", i)
