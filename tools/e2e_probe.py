import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from paper_2508_12093_b200 import hestat as H
from paper_2508_12093_b200 import workloads as W
H.init(0)
S=32768
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
hx = torch.from_numpy(np.ascontiguousarray(x)).pin_memory(); xin = hx.numpy()
hz = torch.empty(S, dtype=torch.float64).pin_memory(); zout = hz.numpy()
for _ in range(20):
    H.decode_column(ctx, H.znorm(ctx, H.encode_column(ctx, xin), 100.0), out=zout)
H.sync()
N=200
t=[0,0,0]
for _ in range(N):
    t0=time.perf_counter(); col=H.encode_column(ctx, xin); t1=time.perf_counter()
    zc=H.znorm(ctx, col, 100.0); t2=time.perf_counter()
    H.decode_column(ctx, zc, out=zout); t3=time.perf_counter()
    t[0]+=t1-t0; t[1]+=t2-t1; t[2]+=t3-t2
print("encode %.1f us, znorm(enqueue) %.1f us, decode(incl wait) %.1f us, total %.1f" % tuple([1e6*v/N for v in t]+[1e6*sum(t)/N]))
# pieces
from paper_2508_12093_b200 import _abi
import ctypes as C
L=_abi.lib()
t0=time.perf_counter()
for _ in range(N): L.hs_sync()
print("bare hs_sync %.1f us" % (1e6*(time.perf_counter()-t0)/N))
col=H.encode_column(ctx, xin)
zc=H.znorm(ctx, col, 100.0); H.sync()
t0=time.perf_counter()
for _ in range(N): H.decode_column(ctx, zc, out=zout)
print("decode only (idle device) %.1f us" % (1e6*(time.perf_counter()-t0)/N))
t0=time.perf_counter()
for _ in range(N): c=H.encode_column(ctx, xin)
print("encode only %.1f us" % (1e6*(time.perf_counter()-t0)/N))
t0=time.perf_counter()
for _ in range(N): zc=H.znorm(ctx, col, 100.0)
H.sync()
print("znorm only loop %.1f us" % (1e6*(time.perf_counter()-t0)/N))
# pipelined: encode step k+1 while step k computes
t = [0, 0, 0]
col = H.encode_column(ctx, xin)
for k in range(N):
    t0 = time.perf_counter(); zc = H.znorm(ctx, col, 100.0); t1 = time.perf_counter()
    col = H.encode_column(ctx, xin); t2 = time.perf_counter()
    H.decode_column(ctx, zc, out=zout); t3 = time.perf_counter()
    t[0] += t1 - t0; t[1] += t2 - t1; t[2] += t3 - t2
print("pipelined: znorm(enqueue) %.1f us, encode next %.1f us, decode %.1f us, total %.1f" % tuple([1e6*v/N for v in t]+[1e6*sum(t)/N]))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for k in range(N):
    zc = H.znorm(ctx, col, 100.0); col = H.encode_column(ctx, xin); H.decode_column(ctx, zc, out=zout)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
