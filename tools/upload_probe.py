"""Dev probe (GPU): cost breakdown of tensor_from_host for a pinned 800 KB array."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
sf.init_runtime(sf.RuntimeOptions())
B = 100000
x_np = torch.zeros(B * 2, dtype=torch.float32).pin_memory().numpy()
def t(name, f, n=200):
    for _ in range(10): f()
    _native.sync(0); s = time.perf_counter()
    for _ in range(n): f()
    _native.sync(0)
    print(f"{name:28s} {(time.perf_counter() - s) / n * 1e6:7.1f} us")
t("device_count", _native.device_count)
t("alloc", lambda: _native.alloc(0, x_np.nbytes))
t("upload", lambda: _native.upload(0, x_np))
t("tensor_from_host", lambda: sf.tensor_from_host(x_np, (B, 2), sf.float32))
xt = torch.from_numpy(x_np); d = torch.empty(B * 2, device="cuda")
t("torch copy_ + sync", lambda: (d.copy_(xt, non_blocking=True), torch.cuda.synchronize()))
buf = _native.alloc(0, x_np.nbytes)
p = x_np.ctypes.data
t("sf_memcpy_h2d pinned", lambda: _native._lib.sf_memcpy_h2d(0, buf.ptr, p, x_np.nbytes))
pg = np.zeros(B * 2, np.float32); pp = pg.ctypes.data
t("sf_memcpy_h2d pageable", lambda: _native._lib.sf_memcpy_h2d(0, buf.ptr, pp, pg.nbytes))
t("sf_memcpy_h2d pageable+sync", lambda: (_native._lib.sf_memcpy_h2d(0, buf.ptr, pp, pg.nbytes), _native.sync(0)))
t("sync only", lambda: _native.sync(0))
import ctypes
rt = ctypes.CDLL("libcudart.so.12") if False else None
s2 = torch.cuda.Stream()
def tc2():
    with torch.cuda.stream(s2):
        d.copy_(xt, non_blocking=True)
    s2.synchronize()
t("torch side stream copy", tc2)
