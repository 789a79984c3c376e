"""Python-side cost of the e2e loop: wrapper calls vs raw C-ABI calls, with/without torch."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "torch":
    import torch  # noqa: F401
    torch.cuda.init()
from paper_2508_12093_b200 import hestat as H, _abi
from paper_2508_12093_b200 import workloads as W
H.init(0)
S = 32768
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
cr = C.CDLL("libcudart.so.12") if False else None
ctx = H.EvalContext(H.CkksParams(slot_count=S))
L = _abi.lib()
# pinned buffers through the library-independent cudart of the process
rt = C.CDLL(os.path.join(os.path.dirname(_abi.LIB_PATH), "libhestat_gpu.so"))
px, pz = C.c_void_p(), C.c_void_p()
cudart = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = C.CDLL(name)
        break
    except OSError:
        pass
assert cudart.cudaHostAlloc(C.byref(px), S * 8, 0) == 0 and cudart.cudaHostAlloc(C.byref(pz), S * 8, 0) == 0
xin = np.ctypeslib.as_array(C.cast(px, C.POINTER(C.c_double)), (S,))
zout = np.ctypeslib.as_array(C.cast(pz, C.POINTER(C.c_double)), (S,))
xin[:] = x
flags = C.c_uint(0)
cudart.cudaGetDeviceFlags(C.byref(flags))
print("device flags", hex(flags.value))
N = 1000
def wrapped():
    col = H.encode_column(ctx, xin)
    for k in range(N):
        zc = H.znorm(ctx, col, 100.0)
        col = H.encode_column(ctx, xin)
        H.decode_column(ctx, zc, out=zout)
for rep in range(2):
    t0 = time.perf_counter(); wrapped(); print("wrapped pipelined %.1f us/step" % (1e6 * (time.perf_counter() - t0) / N))
cfg = H._cfg(None)
enc = L.hs_encode_column; zn = L.hs_znorm; dec = L.hs_decode_column; rel = L.hs_ct_release
xp = H._dp(xin); zp = H._dp(zout)
def raw():
    a = (C.c_void_p * 1)(); n = C.c_uint64(0); o = (C.c_void_p * 1)()
    enc(ctx._h, xp, S, a, C.byref(n))
    for k in range(N):
        col = _abi.hs_column(C.cast(a, C.POINTER(C.c_void_p)), 1, S)
        zn(ctx._h, C.byref(col), 100.0, cfg, o)
        b = (C.c_void_p * 1)()
        enc(ctx._h, xp, S, b, C.byref(n))
        zc = _abi.hs_column(C.cast(o, C.POINTER(C.c_void_p)), 1, S)
        dec(ctx._h, C.byref(zc), zp)
        rel(C.c_void_p(a[0])); rel(C.c_void_p(o[0]))
        a = b
for rep in range(2):
    t0 = time.perf_counter(); raw(); print("raw pipelined %.1f us/step" % (1e6 * (time.perf_counter() - t0) / N))
