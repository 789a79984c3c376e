"""Profiling driver (run under ncu on the GPU box): a few C2 znorm calls."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2508_12093_b200 import hestat as H
from paper_2508_12093_b200 import workloads as W
H.init(0)
x = W.normal(H.synthetic_uniform, 21, 32768, 50.0, 10.0)
ctx = H.EvalContext(H.CkksParams(slot_count=32768))
col = H.encode_column(ctx, x)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    z = H.znorm(ctx, col, 100.0)
H.sync()
import ctypes
from paper_2508_12093_b200 import _abi
for k in range(4):
    r = ctypes.c_double(0); _abi.lib().hs_diag_fp64_rate(k, ctypes.byref(r)); print("fp64 rate kind", k, r.value / 1e12, "T/s")
