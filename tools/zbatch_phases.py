import ctypes as C, os, sys
sys.path[:0]=['.','tests']
from paper_2508_12093_b200 import _abi
_abi.LIB_PATH = os.path.abspath('tools/libhestat_tim.so')
import numpy as np
from paper_2508_12093_b200 import hestat as H, workloads as W
H.init(0)
S=32768
x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=S))
pool=[H.encode_column(ctx, np.roll(x, 97*i)) for i in range(64)]
L=_abi.lib()
for K in (1, 8, 64):
    for _ in range(3): H.znorm_batch(ctx, pool[:K], 100.0)
    H.sync()
    t=(C.c_ulonglong*8)(); L.hs_debug_stat_times(t); v=[t[i] for i in range(8)]
    print(f"K={K}: phaseA {v[1]-v[0]} ns, barrier+totals {v[2]-v[1]} ns, phaseC {v[3]-v[2]} ns, epilogue {v[4]-v[3]} ns")
