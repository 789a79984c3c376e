"""RNS-CKKS Z-score of 1M samples (31 ciphertext chunks of 2^15 slots: the paper's Z-score size)
through the reference's DAG on Tier-R kernels; decrypted output vs the reference's (oracle) output."""
import os, sys, time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np
from oracle_abi import Params, ST_ZNORM, oracle
from paper_2508_12093_b200 import hestat as H, rns as R
S, n = 32768, 1_000_000
x = np.random.default_rng(7).uniform(0.0, 100.0, n)   # the paper's Z-score input range [0, 100], B = 100
L = 25
ctx = R.RnsContext(R.RnsSpec(logN=16, L=L, K=(L + 3) // 3 + 1, dnum=3, logq0=61, logq=60, logp=61, seed=5, h=192))
ev = R.RnsEval(ctx, H.CkksParams(slot_count=S))
ev.stat(R.ZNORM, x[:S], 100.0)  # keys and plans
ws = []
for _ in range(2):
    ev.reset_meter()
    t0 = time.perf_counter()
    z, _ = ev.stat(R.ZNORM, x, 100.0)
    ws.append(time.perf_counter() - t0)
m = ev.meter()
t0 = time.perf_counter()
ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, 100.0)
tcpu = time.perf_counter() - t0
plain = (x - x.mean()) / x.std()
print({"samples": n, "chunks": -(-n // S), "L": L, "wall_s": round(min(ws), 3),
       "rel_err_vs_reference": float(np.max(np.abs(z - ref.out)) / np.max(np.abs(ref.out))),
       "mre_vs_plain": float(np.mean(np.abs(z - plain) / np.maximum(np.abs(plain), 1e-12))),
       "meter": (m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap), "meter_equal": (m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap) == ref.meter,
       "reference_emulator_cpu_s_1core": round(tcpu, 3)})
