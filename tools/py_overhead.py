"""Per-call Python overhead of the e2e wrappers (encode_column / znorm / decode_column) vs the raw C ABI
calls they make, in the pipelined e2e loop (run on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
from paper_2508_12093_b200 import hestat as H, _abi, workloads as W
H.init(0)
S = 32768
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
hx = torch.from_numpy(np.ascontiguousarray(x)).pin_memory(); xin = hx.numpy()
hz = torch.empty(S, dtype=torch.float64).pin_memory(); zout = hz.numpy()
N = 2000
def pipelined(enc, zn, dec):
    col = enc()
    t = [0.0, 0.0, 0.0]
    for k in range(N):
        a = time.perf_counter(); zc = zn(col); b = time.perf_counter()
        col = enc(); c = time.perf_counter()
        dec(zc); d = time.perf_counter()
        t[0] += b - a; t[1] += c - b; t[2] += d - c
    return [1e6 * v / N for v in t]
wr = (lambda: H.encode_column(ctx, xin), lambda col: H.znorm(ctx, col, 100.0), lambda zc: H.decode_column(ctx, zc, out=zout))
L = _abi.lib()
cfg = H._cfg(None)
xp, zp = H._dp(xin), H._dp(zout)
class RawCol:
    __slots__ = ("h", "c")
def r_enc():
    a = (C.c_void_p * 1)(); n = C.c_uint64(0)
    L.hs_encode_column(ctx._h, xp, S, a, C.byref(n))
    r = RawCol(); r.h = a; r.c = _abi.hs_column(C.cast(a, C.POINTER(C.c_void_p)), 1, S); return r
def r_zn(col):
    o = (C.c_void_p * 1)()
    L.hs_znorm(ctx._h, C.byref(col.c), 100.0, cfg, o)
    L.hs_ct_release(C.c_void_p(col.h[0]))
    r = RawCol(); r.h = o; r.c = _abi.hs_column(C.cast(o, C.POINTER(C.c_void_p)), 1, S); return r
def r_dec(zc):
    L.hs_decode_column(ctx._h, C.byref(zc.c), zp)
    L.hs_ct_release(C.c_void_p(zc.h[0]))
for rep in range(3):
    print("wrapped  znorm %.1f encode %.1f decode %.1f" % tuple(pipelined(*wr)))
    print("raw      znorm %.1f encode %.1f decode %.1f" % tuple(pipelined(r_enc, r_zn, r_dec)))
