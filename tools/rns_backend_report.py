"""The BASELINE configs on RNS-backed EvalContexts (the reference's operator surface over
RNS-CKKS) against the reference's decrypted outputs (C oracle, same inputs).

  python tools/rns_backend_report.py [--boot refresh|logical] [--configs C2,C3,C4,C1] [--reps 2]
One JSON line per config case: relative error vs the reference and vs plain fp64, meter /
level equality, wall ms (keys warm, encrypt + statistic + decrypt) and the GPU span of the
statistic (CUDA events on the library stream; host work of the DAG -- refresh decryptions,
ledger -- included), plus the parameter set and its logQP.
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_abi import Cfg, Params, ST_KURT, ST_PEARSON, ST_SKEW, ST_ZNORM, oracle  # noqa: E402
from paper_2508_12093_b200 import _abi  # noqa: E402
from paper_2508_12093_b200 import hestat as H  # noqa: E402
from paper_2508_12093_b200 import workloads as W  # noqa: E402


def plain_value(which, x, y=None):
    xc = x - x.mean()
    if which == ST_KURT:
        return np.mean(xc ** 4) / x.var() ** 2
    if which == ST_SKEW:
        return np.mean(xc ** 3) / x.var() ** 1.5
    if which == ST_PEARSON:
        return np.corrcoef(x, y)[0, 1]
    raise ValueError(which)


class Timer:
    def __init__(self):
        import torch
        self.torch = torch
        self.s = torch.cuda.ExternalStream(_abi.lib().hs_stream())

    def __enter__(self):
        H.sync()
        self.e0 = self.torch.cuda.Event(enable_timing=True)
        self.e1 = self.torch.cuda.Event(enable_timing=True)
        self.t0 = time.perf_counter()
        self.e0.record(self.s)
        return self

    def __exit__(self, *a):
        self.e1.record(self.s)
        self.e1.synchronize()
        self.wall_ms = 1e3 * (time.perf_counter() - self.t0)
        self.gpu_ms = self.e0.elapsed_time(self.e1)


def run(ctx, key, reps):
    spec = W.CONFIG_CASES[key]
    x, y = W.make_inputs(spec, H.synthetic_uniform)
    kw = spec["kwargs"]
    S = spec["params"]["slot_count"]
    best = None
    for _ in range(reps):
        ctx.set_meter(H.CostMeter())
        with Timer() as t:
            if spec["api"] == "invroot":
                cf = kw["cfg"]
                r = H.crypto_invsqrt(ctx, ctx.encrypt(x), kw["S"],
                                     H.InvRootConfig(cheb_degree=cf["cheb_degree"], newton_iters=cf["newton_iters"]),
                                     kw["n_valid"])
                out = ctx.decrypt(r, len(x))
                lvl = r.level()
            elif kw["which"] == ST_ZNORM:
                zc = H.znorm(ctx, H.encode_column(ctx, x), kw["B"])
                out = H.decode_column(ctx, zc)
                lvl = zc.chunks[0].level() if hasattr(zc, "chunks") else None
            else:
                col = H.encode_column(ctx, x)
                if kw["which"] == ST_PEARSON:
                    r = H.pearson(ctx, col, H.encode_column(ctx, y), kw["B"])
                else:
                    r = (H.kurtosis if kw["which"] == ST_KURT else H.skewness)(ctx, col, kw["B"])
                out = ctx.decrypt(r, 1)
                lvl = r.level()
        if best is None or t.wall_ms < best[0]:
            best = (t.wall_ms, t.gpu_ms, out, lvl, ctx.meter().as_tuple())
    wall, gpu, out, lvl, meter = best
    if spec["api"] == "invroot":
        cf = kw["cfg"]
        ref = oracle().invroot(Params(slot_count=S), 0, x, 11, kw["S"], Cfg(cheb_degree=cf["cheb_degree"],
                                                                          newton_iters=cf["newton_iters"]))
        err = float(np.max(np.abs(out - ref.out[:len(x)]) / np.abs(ref.out[:len(x)])))
        err_plain = float(np.max(np.abs(out - 1 / np.sqrt(x * kw["S"])) * np.sqrt(x * kw["S"])))
    else:
        ref = oracle().stat(Params(slot_count=S), kw["which"], x, kw["B"], y=y)
        if kw["which"] == ST_ZNORM:
            err = float(np.max(np.abs(out - ref.out)) / np.max(np.abs(ref.out)))
            p = (x - x.mean()) / x.std()
            err_plain = float(np.max(np.abs(out - p)) / np.max(np.abs(p)))
        else:
            err = float(abs(out[0] - ref.out[0]) / abs(ref.out[0]))
            pv = plain_value(kw["which"], x, y)
            err_plain = float(abs(out[0] - pv) / abs(pv))
    return {"case": key, "rel_err_vs_reference": err, "rel_err_vs_plain_fp64": err_plain,
            "meter_equal": tuple(meter) == tuple(ref.meter),
            "level_equal": lvl is None or lvl == ref.levels[0], "wall_ms": round(wall, 2), "gpu_span_ms": round(gpu, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--boot", default="refresh", choices=["refresh", "logical"])
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    boot = H.BOOT_REFRESH if a.boot == "refresh" else H.BOOT_LOGICAL
    groups = a.configs.split(",")
    ctxs = {}
    for key in W.CONFIG_CASES:
        if key.split("_")[0] not in groups:
            continue
        S = W.CONFIG_CASES[key]["params"]["slot_count"]
        if S not in ctxs:
            ctxs[S] = H.EvalContext(H.CkksParams(slot_count=S), rng_seed=7, backend="rns", boot=boot)
            sp, _ = ctxs[S].rns_spec()
            logqp = sp.logq0 + sp.L * sp.logq + sp.K * sp.logp
            print(json.dumps({"params": {"slot_count": S, "logN": sp.logN, "L": sp.L, "K": sp.K, "dnum": sp.dnum,
                                         "logq0": sp.logq0, "logq": sp.logq, "logp": sp.logp, "h": sp.h,
                                         "logQP_bits": logqp, "boot": a.boot,
                                         "security": ("inside the 128-bit budget (HE standard, N=2^%d: %d bits)"
                                                      % (sp.logN, {13: 218, 14: 438, 15: 881, 16: 1761}
                                                         .get(sp.logN, 0)))
                                         if logqp <= {13: 218, 14: 438, 15: 881, 16: 1761}.get(sp.logN, 0)
                                         else "functional, not 128-bit"}}), flush=True)
        print(json.dumps(run(ctxs[S], key, a.reps)), flush=True)


if __name__ == "__main__":
    main()
