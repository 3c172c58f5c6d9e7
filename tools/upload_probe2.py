"""Dev probe (GPU): why upload() is slower than a bare sf_memcpy_h2d."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1903_01855_b200 as sf
from paper_1903_01855_b200 import _native
sf.init_runtime(sf.RuntimeOptions())
B = 100000
x_np = torch.zeros(B * 2, dtype=torch.float32).pin_memory().numpy()
L = _native._lib
def t(name, f, n=200):
    for _ in range(10): f()
    _native.sync(0); s = time.perf_counter()
    for _ in range(n): f()
    _native.sync(0)
    print(f"{name:28s} {(time.perf_counter() - s) / n * 1e6:7.1f} us")
a = np.ascontiguousarray(x_np)
print("same obj", a is x_np, a.ctypes.data == x_np.ctypes.data)
def manual():
    b = _native.alloc(0, x_np.nbytes)
    L.sf_memcpy_h2d(0, b.ptr, x_np.ctypes.data, x_np.nbytes)
    return b
t("manual alloc+h2d", manual)
keep = []
def manual_keep():
    b = _native.alloc(0, x_np.nbytes)
    L.sf_memcpy_h2d(0, b.ptr, x_np.ctypes.data, x_np.nbytes)
    keep.append(b)
    if len(keep) > 4: keep.pop(0)
t("manual alloc+h2d keep4", manual_keep)
t("upload", lambda: _native.upload(0, x_np))
bb = _native.alloc(0, x_np.nbytes)
t("h2d fixed dst", lambda: L.sf_memcpy_h2d(0, bb.ptr, x_np.ctypes.data, x_np.nbytes))
t("upload again", lambda: _native.upload(0, x_np))
