"""Phase timestamps of the statistics kernel (block 0, %globaltimer) from a
-DHS_STAT_TIMING build of the library (tools/libhestat_tim.so)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_12093_b200 import _abi  # noqa: E402
_abi.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhestat_tim.so")
import numpy as np  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402

H.init(0)
L = _abi.lib()
for S in (1024, 32768):
    x = W.normal(H.synthetic_uniform, 21, S, 50.0, 10.0)
    ctx = H.EvalContext(H.CkksParams(slot_count=S))
    col = H.encode_column(ctx, x)
    for name, fn in (("znorm", lambda: H.znorm(ctx, col, 100.0)), ("moments", lambda: H.moments(ctx, col, 100.0))):
        for _ in range(5):
            fn()
        H.sync()
        t = (C.c_ulonglong * 8)()
        L.hs_debug_stat_times(t)
        v = [t[i] for i in range(8)]
        print(f"S={S} {name}: start->A {v[1]-v[0]} ns, terms+blockred {v[5]-v[1]} ns, grid.sync {v[6]-v[5]} ns, "
              f"partials {v[7]-v[6]} ns, ->C {v[3]-v[7]} ns, C {v[4]-v[3]} ns")
