"""RNS ZNorm (L=25) time and accuracy versus the key-switching decomposition (dnum, K)."""
import os, sys, time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np
from oracle_abi import Params, ST_ZNORM, oracle
from paper_2508_12093_b200 import hestat as H, rns as R, workloads as W
S, L = 32768, 25
x = W.normal(H.synthetic_uniform, 42, S, 50.0, 10.0)
ref = oracle().stat(Params(slot_count=S), ST_ZNORM, x, 100.0)
for dnum in (1, 2, 3, 4, 6):
    alpha = -(-(L + 1) // dnum)
    K = -(-(61 + (alpha - 1) * 60) // 61) + 1
    try:
        ctx = R.RnsContext(R.RnsSpec(logN=16, L=L, K=K, dnum=dnum, logq0=61, logq=60, logp=61, seed=5, h=192))
        ev = R.RnsEval(ctx, H.CkksParams(slot_count=S))
        ev.stat(R.ZNORM, x, 100.0)
        ws = []
        for _ in range(3):
            t0 = time.perf_counter(); z, _ = ev.stat(R.ZNORM, x, 100.0); ws.append(time.perf_counter() - t0)
        print(dnum, alpha, K, "ms", round(1e3 * min(ws), 1), "err", float(np.max(np.abs(z - ref.out)) / np.max(np.abs(ref.out))), flush=True)
        ev.close(); ctx.close()
    except Exception as e:
        print(dnum, alpha, K, "failed", type(e).__name__, str(e)[:120], flush=True)
