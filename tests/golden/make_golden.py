"""Generate tests/golden/golden_small.npz from the COMPILED REFERENCE.

Run in the build container (where /root/reference exists and oracle/Makefile
built oracle/_ref/libhestat_ref.so):

    python tests/golden/make_golden.py

Every case stores its inputs, so replays never regenerate data: the C
restatement (tests/test_oracle.py, CPU) and the CUDA product
(tests/test_parity_golden.py, GPU) are both checked bitwise against the
reference's own outputs, status codes, levels and meters.

Large config-shaped workloads (32768 slots) are stored as SHA-256 digests of the
output bit patterns plus meters/levels (tests/golden/golden_configs.json), with
inputs regenerated from seeds by paper_2508_12093_b200.workloads.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from golden_io import run_case  # noqa: E402
from oracle_abi import (ALL_SLOTS, FIT_COS2, FIT_EXP, FIT_IDENT, FIT_INVSQRT_SHIFTED,  # noqa: E402
                        FIT_RECIP2, FIT_SQRT_SHIFTED, FIT_SQUARE, Cfg, Params, reference)


def golden_cases():
    """Deterministic case list: (name, api, params, kwargs).  Inputs come from
    numpy's PCG64 uniform stream only (platform-stable)."""
    rng = np.random.default_rng(20260811)
    cases = []

    def P(**kw):
        return Params(**kw)

    # --- ckks.hpp ops (KATs of ckks_test.cpp + randomized) ------------------
    kat4 = P(slot_count=4, quantize=False, auto_bootstrap=False)
    cases.append(("kat_add", "op", kat4, dict(op=0, a=[1, 2, 0, 0], la=11, b=[3, 4, 0, 0], lb=11)))
    cases.append(("kat_sub", "op", kat4, dict(op=1, a=[3, 4, 0, 0], la=11, b=[1, 1, 0, 0], lb=11)))
    cases.append(("kat_mul", "op", kat4, dict(op=3, a=[1, 2, 0, 0], la=11, b=[3, 4, 0, 0], lb=11)))
    cases.append(("kat_rot1", "op", kat4, dict(op=6, a=[1, 2, 3, 4], la=11, k=1)))
    cases.append(("kat_rotm1", "op", kat4, dict(op=6, a=[1, 2, 3, 4], la=11, k=-1)))
    cases.append(("kat_rot5", "op", kat4, dict(op=6, a=[1, 2, 3, 4], la=11, k=5)))
    cases.append(("kat_mulpt_vec", "op", kat4, dict(op=5, a=[2, 4, 0, 0], la=11, vec=[1, 0, 1, 0])))
    cases.append(("kat_mulpt_badvec", "op", kat4, dict(op=5, a=[2, 4, 0, 0], la=11, vec=[1, 2])))
    cases.append(("kat_mul_exhausted", "op", kat4, dict(op=3, a=[1, 0, 0, 0], la=0, b=[1, 0, 0, 0], lb=0)))
    cases.append(("kat_mulpt_exhausted", "op", kat4, dict(op=4, a=[1, 0, 0, 0], la=0, c=2.0)))
    cases.append(("kat_sum3", "op", kat4, dict(op=8, a=[1, 2, 3, 0], la=11, n_valid=3)))
    cases.append(("kat_sum_dirty", "op", P(slot_count=4, quantize=False, auto_bootstrap=False, debug_checks=True),
                  dict(op=8, a=[1, 2, 3, 4], la=11, n_valid=3)))
    cases.append(("kat_autoboot", "op", P(slot_count=4, quantize=False), dict(op=3, a=[2, 0, 0, 0], la=0, b=[2, 0, 0, 0], lb=0)))
    cases.append(("kat_shape", "op", kat4, dict(op=0, a=[1, 2, 3], la=11, b=[1, 2, 3, 4], lb=11)))
    for q in (True, False):
        for S in (8, 64, 256):
            a = rng.uniform(-100, 100, S)
            b = rng.uniform(-100, 100, S)
            vec = rng.uniform(-2, 2, S)
            for op in range(9):
                for la, lb in ((11, 11), (0, 4), (5, 0)):
                    cases.append((f"op{op}_S{S}_q{int(q)}_l{la}{lb}", "op", P(slot_count=S, quantize=q),
                                  dict(op=op, a=a, la=la, b=b, lb=lb, c=float(rng.uniform(-3, 3)), vec=vec,
                                       k=int(rng.integers(-3 * S, 3 * S)), n_valid=S)))
    # unquantized-input bootstrap (Ciphertext(vector, level) with raw values)
    raw = rng.uniform(-1, 1, 64)
    cases.append(("boot_raw_q", "op", P(slot_count=64), dict(op=7, a=raw, la=0)))
    cases.append(("mul_autoboot_raw_q", "op", P(slot_count=64), dict(op=3, a=raw, la=0, b=raw[::-1].copy(), lb=3)))
    # quantisation range: large magnitudes / subnormal products / signed zeros
    big = np.concatenate([rng.uniform(-1e6, 1e6, 16), [0.0, -0.0, 1e-300, -1e-300, 5e-13, -5e-13, 2.0 ** -41, -(2.0 ** -41),
                                                         3 * 2.0 ** -41, 2047.9999, -2048.0, 4096.5, 1e15, -1e15, 2 ** 52, -(2 ** 53)]])
    big = np.concatenate([big, np.zeros(64 - len(big))])
    for op in (0, 2, 3, 4, 7):
        cases.append((f"edge_op{op}", "op", P(slot_count=64), dict(op=op, a=big, la=11, b=big[::-1].copy(), lb=11,
                                                                      c=-0.0 if op == 4 else 1e-3)))

    # --- chebyshev.hpp ------------------------------------------------------
    for kind, S, deg in [(FIT_IDENT, 1, 3), (FIT_SQUARE, 1, 2), (FIT_EXP, 1, 63), (FIT_INVSQRT_SHIFTED, 100.0, 511),
                         (FIT_INVSQRT_SHIFTED, 400.0, 15), (FIT_SQRT_SHIFTED, 20.0, 511), (FIT_RECIP2, 1, 1023),
                         (FIT_COS2, 1, 255), (FIT_EXP, 1, 0)]:
        cases.append((f"fit_{kind}_{deg}", "fit", None, dict(kind=kind, S=S, degree=deg, lo=-1.0, hi=1.0)))
    cases.append(("fit_dom", "fit", None, dict(kind=FIT_SQUARE, S=1, degree=4, lo=0.0, hi=2.0)))
    x64 = rng.uniform(-1, 1, 64)
    for q in (True, False):
        for deg in (0, 1, 2, 3, 5, 7, 12, 15, 31, 63, 100, 127, 255, 511, 1023):
            cf = rng.uniform(-1, 1, deg + 1) / np.sqrt(deg + 1.0)
            cases.append((f"eval_d{deg}_q{int(q)}", "eval_encrypted", P(slot_count=64, quantize=q),
                          dict(coeffs=cf, lo=-1.0, hi=1.0, x=x64, lx=11)))
        cf = rng.uniform(-1, 1, 16)
        cases.append((f"eval_dom_q{int(q)}", "eval_encrypted", P(slot_count=64, quantize=q),
                      dict(coeffs=cf, lo=0.0, hi=2.0, x=x64 + 1.0, lx=11)))
        cases.append((f"eval_short_q{int(q)}", "eval_encrypted", P(slot_count=64, quantize=q),
                      dict(coeffs=rng.uniform(-1, 1, 256), lo=-1.0, hi=1.0, x=x64, lx=3)))
        cases.append((f"eval_deep_q{int(q)}", "eval_encrypted", P(slot_count=64, quantize=q, max_level=5),
                      dict(coeffs=rng.uniform(-1, 1, 128), lo=-1.0, hi=1.0, x=x64, lx=5)))
    cases.append(("eval_domain_viol", "eval_encrypted", P(slot_count=8, quantize=False, debug_checks=True),
                  dict(coeffs=[0, 1, 0, 0], lo=-1.0, hi=1.0, x=[1.5] + [0] * 7, lx=11)))
    cases.append(("eval_noauto", "eval_encrypted", P(slot_count=8, auto_bootstrap=False),
                  dict(coeffs=rng.uniform(-1, 1, 32), lo=-1.0, hi=1.0, x=x64[:8], lx=2)))

    # --- primitives.hpp -----------------------------------------------------
    p64 = P(slot_count=64, quantize=False)
    cases.append(("newton_fixed", "newton_refine", P(slot_count=4, quantize=False),
                  dict(x=[1, 0, 0, 0], lx=11, y0=[1, 0, 0, 0], ly=11, n=2, iters=3, n_valid=ALL_SLOTS)))
    cases.append(("newton_isqrt", "newton_refine", P(slot_count=4, quantize=False),
                  dict(x=[0.25, 0, 0, 0], lx=11, y0=[1.8, 0, 0, 0], ly=11, n=2, iters=4, n_valid=ALL_SLOTS)))
    cases.append(("newton_inv", "newton_refine", P(slot_count=4, quantize=False),
                  dict(x=[2.0, 0, 0, 0], lx=11, y0=[0.7, 0, 0, 0], ly=11, n=1, iters=5, n_valid=ALL_SLOTS)))
    cases.append(("newton_diverge", "newton_refine", P(slot_count=4, quantize=False, debug_checks=True),
                  dict(x=[1, 0, 0, 0], lx=11, y0=[1e3, 0, 0, 0], ly=11, n=2, iters=6, n_valid=1)))
    xt = rng.uniform(0.2, 3.0, 64)
    for q in (True, False):
        for n in (1, 2, 3, 4):
            cases.append((f"newton_n{n}_q{int(q)}", "newton_refine", P(slot_count=64, quantize=q),
                          dict(x=xt, lx=7, y0=1.0 / np.sqrt(xt) * 1.2, ly=3, n=n, iters=5, n_valid=ALL_SLOTS)))
    grid = np.linspace(0.001, 100.0, 256) / 100.0
    for q in (True, False):
        for which in range(4):
            for cfg in (Cfg(), Cfg(cheb_degree=15, newton_iters=2), Cfg(baseline_mode=True), Cfg(n=1, newton_iters=0),
                        Cfg(cheb_degree=255, newton_iters=4, baseline_mode=True, baseline_iters=9)):
                cases.append((f"invroot{which}_q{int(q)}_{cfg.cheb_degree}_{cfg.newton_iters}_{int(cfg.baseline_mode)}_{cfg.n}",
                              "invroot", P(slot_count=256, quantize=q, debug_checks=True),
                              dict(which=which, x=grid, lx=11, S=100.0, cfg=cfg, n_valid=ALL_SLOTS)))
    cases.append(("invsqrt_known", "invroot", P(slot_count=16, quantize=False),
                  dict(which=0, x=[0.01, 0.04] + [0.5] * 14, lx=11, S=100.0, cfg=Cfg(), n_valid=2)))
    cases.append(("invsqrt_domain", "invroot", P(slot_count=8, quantize=False, debug_checks=True),
                  dict(which=0, x=[2.5] + [0.5] * 7, lx=11, S=10.0, cfg=Cfg(), n_valid=1)))
    cases.append(("invsqrt_zero", "invroot", P(slot_count=8, quantize=False, debug_checks=True),
                  dict(which=0, x=[0.0] + [0.5] * 7, lx=11, S=10.0, cfg=Cfg(), n_valid=1)))
    cases.append(("invsqrt_noauto", "invroot", P(slot_count=8, quantize=False, auto_bootstrap=False),
                  dict(which=0, x=[0.5] * 8, lx=11, S=1.0, cfg=Cfg(), n_valid=1)))
    cases.append(("invsqrt_badcfg", "invroot", P(slot_count=8), dict(which=0, x=[0.5] * 8, lx=11, S=1.0, cfg=Cfg(n=3), n_valid=1)))
    cases.append(("invsqrt_badS", "invroot", P(slot_count=8), dict(which=0, x=[0.5] * 8, lx=11, S=-1.0, cfg=Cfg(), n_valid=1)))
    cases.append(("sqrt_known", "invroot", P(slot_count=16, quantize=False),
                  dict(which=3, x=[0.2, 0.0, 1.0] + [0.5] * 13, lx=11, S=20.0, cfg=Cfg(), n_valid=3)))
    sv = np.concatenate([[0.0, 0.5, -0.3, 0.08, 0.9, -0.9, 1.0, -1.0], rng.uniform(-1, 1, 56)])
    for q in (True, False):
        cases.append((f"sign_g3_q{int(q)}", "crypto_sign", P(slot_count=64, quantize=q), dict(x=sv, lx=11, mode=0, folds=7, polys=[])))
        cases.append((f"sign_g3_8_q{int(q)}", "crypto_sign", P(slot_count=64, quantize=q), dict(x=sv, lx=11, mode=0, folds=8, polys=[])))
        cases.append((f"sign_custom_q{int(q)}", "crypto_sign", P(slot_count=64, quantize=q),
                      dict(x=sv, lx=11, mode=1, folds=3, polys=[[0.0, 35 / 16, 0.0, -35 / 16, 0.0, 21 / 16, 0.0, -5 / 16], [0.0, 1.5, 0.0, -0.5]])))
    cases.append(("sign_bad", "crypto_sign", P(slot_count=8), dict(x=[0.5] * 8, lx=11, mode=1, folds=1, polys=[[0.1, 1.0]])))
    cases.append(("sign_domain", "crypto_sign", P(slot_count=8, debug_checks=True), dict(x=[1.5] * 8, lx=11, mode=0, folds=7, polys=[])))

    # --- column.hpp / stats.hpp ---------------------------------------------
    u100 = rng.uniform(0, 100, 1000)
    u20 = rng.uniform(0, 20, 1000)
    v150 = rng.uniform(1, 19, 150)
    y150 = 0.7 * v150 + 0.3 * rng.uniform(1, 19, 150)
    y1000 = 0.6 * u20 + 0.4 * rng.uniform(0, 20, 1000)
    for which in range(9):
        for q, dbg in ((True, True), (False, False)):
            cases.append((f"stat{which}_1000_q{int(q)}", "stat", P(slot_count=1024, quantize=q, debug_checks=dbg),
                          dict(which=which, x=u100, B=100.0 if which != 2 else 10000.0, y=0.5 * u100 + 3.0, cfg=Cfg())))
            cases.append((f"stat{which}_multichunk_q{int(q)}", "stat", P(slot_count=64, quantize=q, debug_checks=dbg),
                          dict(which=which, x=v150, B=20.0, y=y150, cfg=Cfg())))
        cases.append((f"stat{which}_1000_c15", "stat", P(slot_count=1024),
                      dict(which=which, x=u20, B=20.0, y=y1000, cfg=Cfg(cheb_degree=15, newton_iters=2))))
    cases.append(("stat_mean_kat", "stat", P(slot_count=4, quantize=False), dict(which=0, x=[1, 2, 3, 4], B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_var_kat", "stat", P(slot_count=4, quantize=False), dict(which=1, x=[1, 2, 3, 4], B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_skew_spike", "stat", P(slot_count=8, quantize=False), dict(which=6, x=[0, 0, 0, 10], B=5.0, y=None, cfg=Cfg())))
    cases.append(("stat_kurt_2pt", "stat", P(slot_count=16, quantize=False), dict(which=5, x=[-1, 1] * 4, B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_empty", "stat", P(slot_count=8), dict(which=0, x=[], B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_degenerate", "stat", P(slot_count=16, quantize=False, debug_checks=True),
                  dict(which=4, x=[1.0] * 8, B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_nearzero_mean", "stat", P(slot_count=16, quantize=False, debug_checks=True),
                  dict(which=7, x=[-1, 1] * 4, B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_pearson_len", "stat", P(slot_count=16), dict(which=8, x=[1, 2, 3], B=1.0, y=[1, 2], cfg=Cfg())))
    cases.append(("stat_nonfinite", "stat", P(slot_count=16), dict(which=0, x=[1, float("inf")], B=1.0, y=None, cfg=Cfg())))
    cases.append(("stat_badB", "stat", P(slot_count=16), dict(which=0, x=[1, 2], B=0.0, y=None, cfg=Cfg())))
    # magnitudes beyond the exact-sum bound (sum|A| >= 2^52 grid units): the fused
    # reductions must fall back to the literal rotate-and-add butterfly
    vbig = rng.uniform(1e5, 1e6, 60)
    for which in (0, 1, 2, 3, 5, 6, 8):
        cases.append((f"stat{which}_bigsum", "stat", P(slot_count=64),
                      dict(which=which, x=vbig, B=1e-2 if which != 2 else 1e-4, y=vbig[::-1].copy(), cfg=Cfg())))
    return cases


def _enc_kw(kw):
    arrays, scal = {}, {}
    for k, v in kw.items():
        if isinstance(v, Cfg):
            scal[k] = {"__cfg__": vars(v)}
        elif k == "polys":
            scal[k] = [list(map(float, p)) for p in v]
        elif isinstance(v, (list, np.ndarray)) and k not in ("polys",):
            arrays[k] = np.asarray(v, dtype=np.float64)
        else:
            scal[k] = v
    return arrays, scal


def main():
    ref = reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    index, blobs = [], {}
    for name, api, params, kw in golden_cases():
        res = run_case(ref, api, params, kw)
        rc, out, levels, meter = res
        arrays, scal = _enc_kw(kw)
        for k, v in arrays.items():
            blobs[f"{name}/in/{k}"] = v
        blobs[f"{name}/out"] = np.asarray(out, dtype=np.float64)
        index.append(dict(name=name, api=api, params=vars(params) if params else None, arrays=sorted(arrays),
                          scalars=scal, rc=int(rc), levels=[int(x) for x in levels], meter=[int(x) for x in meter],
                          msg=ref.last_error() if rc else ""))
    blobs["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    path = os.path.join(HERE, "golden_small.npz")
    np.savez_compressed(path, **blobs)
    print(f"wrote {len(index)} cases to {path} ({os.path.getsize(path) / 1e3:.0f} kB)")

    # config-shaped digests
    from paper_2508_12093_b200 import workloads as W  # noqa: E402
    cfgs = {}
    for key, spec in W.CONFIG_CASES.items():
        p = Params(**spec["params"])
        x, y = W.make_inputs(spec, ref.synthetic_uniform)
        kw = dict(spec["kwargs"], x=x, y=y)
        kw["cfg"] = Cfg(**kw["cfg"])
        res = run_case(ref, spec["api"], p, kw)
        cfgs[key] = dict(rc=int(res[0]), levels=[int(v) for v in res[2]], meter=[int(v) for v in res[3]],
                         sha256=hashlib.sha256(np.ascontiguousarray(res[1]).view(np.uint64).tobytes()).hexdigest(),
                         head=[float(v) for v in res[1][:4]],
                         input_sha256=hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest())
        print(key, cfgs[key]["meter"], cfgs[key]["levels"], cfgs[key]["head"])
    with open(os.path.join(HERE, "golden_configs.json"), "w") as f:
        json.dump(cfgs, f, indent=1)


if __name__ == "__main__":
    main()
