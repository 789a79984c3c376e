"""Tier-R statistics on real RNS-CKKS ciphertexts vs the reference (oracle) outputs.

  python tools/rns_stats_report.py [--logN 16] [--L 26]
One JSON line per statistic: relative error of the decrypted result against the
reference's output and against plain fp64, meter equality, wall time (keys warm).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_abi import (Params, ST_KURT, ST_MOMENTS, ST_PEARSON, ST_SKEW, ST_ZNORM, oracle)  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import rns as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logN", type=int, default=16)
    ap.add_argument("--L", type=int, default=28)
    ap.add_argument("--logq", type=int, default=60)
    ap.add_argument("--extraK", type=int, default=1)
    ap.add_argument("--h", type=int, default=192)
    ap.add_argument("--logp", type=int, default=61)
    ap.add_argument("--K", type=int, default=0, help="special primes (default: alpha + extraK)")
    a = ap.parse_args()
    S = 1 << (a.logN - 1)
    K = a.K or (a.L + 3) // 3 + a.extraK
    ctx = R.RnsContext(R.RnsSpec(logN=a.logN, L=a.L, K=K, dnum=3, logq0=61, logq=a.logq, logp=a.logp, seed=3, h=a.h))
    ev = R.RnsEval(ctx, H.CkksParams(slot_count=S))
    rng = np.random.default_rng(11)
    x2 = 50 + 10 * rng.standard_normal(S)                 # C2
    x3 = np.exp(0.5 * rng.standard_normal(S))            # C3 log-normal
    z = rng.standard_normal(S)
    x4 = np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(S)
    y4 = np.sqrt(0.6) * z + np.sqrt(0.4) * rng.standard_normal(S)
    cases = [("znorm", R.ZNORM, ST_ZNORM, x2, None, 100.0), ("moments", R.MOMENTS, ST_MOMENTS, x2, None, 100.0),
             ("kurtosis", R.KURTOSIS, ST_KURT, x3, None, 20.0), ("skewness", R.SKEWNESS, ST_SKEW, x3, None, 20.0),
             ("pearson", R.PEARSON, ST_PEARSON, x4, y4, 20.0)]
    ev.stat(R.ZNORM, x2, 100.0)  # warm: keys (relin + 15 rotations), plans
    for name, code, oc, x, y, B in cases:
        ev.reset_meter()
        t0 = time.perf_counter()
        out, lv = ev.stat(code, x, B, y=y, out_n=1)
        wall = time.perf_counter() - t0
        ref = oracle().stat(Params(slot_count=S), oc, x, B, y=y)
        if code == R.ZNORM:
            err = float(np.max(np.abs(out - ref.out)) / np.max(np.abs(ref.out)))
            plain = (x - x.mean()) / x.std()
            err_plain = float(np.max(np.abs(out - plain)) / np.max(np.abs(plain)))
        elif code == R.MOMENTS:
            err = float(max(abs(out[0] - ref.out[0]) / abs(ref.out[0]), abs(out[1] - ref.out[S]) / abs(ref.out[S])))
            err_plain = float(abs(out[1] - x.var() / B ** 2) / (x.var() / B ** 2))
        else:
            err = float(abs(out[0] - ref.out[0]) / abs(ref.out[0]))
            xc = x - x.mean()
            if code == R.KURTOSIS:
                pv = np.mean(xc ** 4) / x.var() ** 2
            elif code == R.SKEWNESS:
                pv = np.mean(xc ** 3) / x.var() ** 1.5
            else:
                pv = np.corrcoef(x, y)[0, 1]
            err_plain = float(abs(out[0] - pv) / abs(pv))
        m = ev.meter()
        print(json.dumps({"stat": name, "logN": a.logN, "L": a.L, "logq": a.logq, "K": K, "h": a.h, "rel_err_vs_reference": err,
                          "rel_err_vs_plain_fp64": err_plain,
                          "meter_equal": (m.mul_ct, m.mul_pt, m.add, m.rotate, m.bootstrap) == ref.meter,
                          "levels_equal": int(lv[0]) == ref.levels[0], "wall_s": round(wall, 4)}), flush=True)


if __name__ == "__main__":
    main()
