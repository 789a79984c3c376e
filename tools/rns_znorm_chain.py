import sys, time, os
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
import numpy as np
from oracle_abi import Params, ST_ZNORM, oracle
from paper_2508_12093_b200 import hestat as H, rns as R, workloads as W
S = 32768
x = W.normal(H.synthetic_uniform, 42, S, 50.0, 10.0)
ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, 100.0)
for L in (28, 26, 25, 24):
    try:
        ctx = R.RnsContext(R.RnsSpec(logN=16, L=L, K=(L + 3) // 3 + 1, dnum=3, logq0=61, logq=60, logp=61, seed=5, h=192))
        ev = R.RnsEval(ctx, H.CkksParams(slot_count=S))
        ev.stat(R.ZNORM, x, 100.0)
        ws = []
        for _ in range(3):
            ev.reset_meter(); t0 = time.perf_counter(); z, _ = ev.stat(R.ZNORM, x, 100.0); ws.append(time.perf_counter() - t0)
        m = ev.meter()
        print(L, "ms", round(1e3 * min(ws), 1), "err", float(np.max(np.abs(z - ref.out)) / np.max(np.abs(ref.out))), (m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap) == ref.meter, flush=True)
        ev.close(); ctx.close()
    except Exception as e:
        print(L, "failed", type(e).__name__, str(e)[:100], flush=True)
