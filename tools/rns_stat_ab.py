"""A/B of the RNS ZNorm time between library builds: HESTAT_LIB=... python tools/rns_stat_ab.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2508_12093_b200 import _abi
if os.environ.get("HESTAT_LIB"):
    _abi.LIB_PATH = os.environ["HESTAT_LIB"]
from paper_2508_12093_b200 import hestat as H, rns as R
L = 25
ctx = R.RnsContext(R.RnsSpec(logN=16, L=L, K=(L + 3) // 3 + 1, dnum=3, logq0=61, logq=60, logp=61, seed=5, h=192))
ev = R.RnsEval(ctx, H.CkksParams(slot_count=32768))
x = 50 + 10 * np.random.default_rng(1).standard_normal(32768)
ev.stat(R.ZNORM, x, 100.0)
ws = []
for _ in range(4):
    t0 = time.perf_counter(); ev.stat(R.ZNORM, x, 100.0); ws.append(time.perf_counter() - t0)
print("znorm L=25 ms", round(1e3 * min(ws), 1))
