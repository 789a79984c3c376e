import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, ctypes as C
from paper_2508_12093_b200 import hestat as H, _abi
from paper_2508_12093_b200 import workloads as W
H.init(0)
S = 32768
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
col = H.encode_column(ctx, x)
L = _abi.lib()
for _ in range(50): H.znorm(ctx, col, 100.0)
H.sync()
N = 400
def loop(f):
    H.sync(); t0 = time.perf_counter()
    for _ in range(N): r = f()
    t1 = time.perf_counter(); H.sync()
    return 1e6 * (t1 - t0) / N
print("H.znorm %.1f us" % loop(lambda: H.znorm(ctx, col, 100.0)))
c, keep = col._c()
arr = (C.c_void_p * 1)()
cfg = H._cfg(None)
def raw():
    L.hs_znorm(ctx._h, C.byref(c), 100.0, cfg, arr)
    L.hs_ct_release(C.c_void_p(arr[0]))
print("raw hs_znorm+release %.1f us" % loop(raw))
print("argtypes", L.hs_znorm.argtypes, L.hs_znorm.restype)
print("col._c %.2f us" % loop(lambda: col._c()))
print("_abi.lib %.2f us" % loop(lambda: _abi.lib()))
P = C.PyDLL(_abi.LIB_PATH)
for name in ("hs_znorm", "hs_ct_release"):
    getattr(P, name).restype = getattr(L, name).restype
    getattr(P, name).argtypes = getattr(L, name).argtypes
def rawp():
    P.hs_znorm(ctx._h, C.byref(c), 100.0, cfg, arr)
    P.hs_ct_release(C.c_void_p(arr[0]))
print("PyDLL raw hs_znorm+release %.1f us" % loop(rawp))
print("CDLL raw again %.1f us" % loop(raw))
print("H.znorm again %.1f us" % loop(lambda: H.znorm(ctx, col, 100.0)))
def raw2():
    L.hs_znorm(ctx._h, C.byref(c), 100.0, cfg, arr)
    return H.EncryptedColumn([H.Ciphertext._own(C.c_void_p(arr[0]))], col.n_valid, col.name)
print("raw + wrap %.1f us" % loop(raw2))
import threading
print("threads", threading.active_count(), [t.name for t in threading.enumerate()])
