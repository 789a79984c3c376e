"""Replay golden / oracle cases through the product (paper_2508_12093_b200.hestat).

Returns the same (rc, out, levels, meter) tuple as tests/oracle_abi.py so a GPU
result can be compared bit-for-bit with the reference's stored outputs and with
the live C oracle.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2508_12093_b200 import hestat as H

CODE = {H.too_many_values: 2, H.level_exhausted: 3, H.length_mismatch: 4, H.dirty_padding: 5,
        H.non_finite_target: 6, H.domain_violation: 7, H.divergence: 8, H.empty_column: 9,
        H.degenerate_variance: 10, H.near_zero_mean: 11, H.io_error: 12, H.missing_column: 13,
        H.unparsable_cell: 14, H.non_finite_value: 15, H.zero_reference: 16}

FIT_TARGETS = {
    2: lambda x: x,
    3: lambda x: x * x,
    4: math.exp,
    5: lambda x: 1.0 / (2.0 + x),
    6: lambda x: math.cos(2 * x),
    7: lambda x: math.cos(3.0 * x),
    8: lambda x: 1.0,
    9: math.sqrt,
}


def params_of(p) -> H.CkksParams:
    return H.CkksParams(slot_count=p.slot_count, max_level=p.max_level, scale_bits=p.scale_bits,
                        quantize=bool(p.quantize), auto_bootstrap=bool(p.auto_bootstrap),
                        debug_checks=bool(p.debug_checks))


def cfg_of(c) -> H.InvRootConfig:
    if c is None:
        return H.InvRootConfig()
    if isinstance(c, dict):
        return H.InvRootConfig(**c)
    return H.InvRootConfig(c.n, c.cheb_degree, c.newton_iters, bool(c.baseline_mode), c.baseline_iters)


def _code(e: Exception) -> int:
    for cls, code in CODE.items():
        if type(e) is cls:
            return code
    if isinstance(e, H.cuda_error):
        raise e
    if isinstance(e, H.error):
        return 1
    raise e


def run_case(api, params, kw):
    """(rc, out, levels, meter) for one case on the GPU product."""
    if api == "fit":
        kind, S, deg = kw["kind"], kw["S"], kw["degree"]
        try:
            if kind in (0, 1):
                f = (lambda t: H.scaled_target(H.ScaledTargetKind(kind), S, t))
            else:
                f = FIT_TARGETS[kind]
            s = H.fit(f, deg, kw["lo"], kw["hi"])
            return 0, np.asarray(s.coeffs), (0,), (0,) * 5
        except H.error as e:
            return _code(e), np.zeros(max(deg + 1, 1)), (0,), (0,) * 5
    ctx = H.EvalContext(params_of(params))
    S = params.slot_count
    levels = [0]
    out = np.zeros(S)
    try:
        if api == "op":
            a = H.Ciphertext(kw["a"], kw["la"])
            b = H.Ciphertext(kw["b"], kw.get("lb", 0)) if kw.get("b") is not None else H.Ciphertext()
            op = kw["op"]
            if op == 0:
                r = ctx.add_ct(a, b)
            elif op == 1:
                r = ctx.sub_ct(a, b)
            elif op == 2:
                r = ctx.add_pt(a, kw.get("c", 0.0))
            elif op == 3:
                r = ctx.mul_ct(a, b)
            elif op == 4:
                r = ctx.mul_pt(a, kw.get("c", 0.0))
            elif op == 5:
                r = ctx.mul_pt(a, np.asarray(kw.get("vec"), dtype=np.float64))
            elif op == 6:
                r = ctx.rotate(a, kw.get("k", 0))
            elif op == 7:
                r = ctx.bootstrap(a)
            else:
                r = ctx.sum_all_slots(a, kw.get("n_valid", 0))
            out, levels = r.slots(), [r.level()]
        elif api == "eval_encrypted":
            s = H.ChebyshevSeries(list(np.asarray(kw["coeffs"], dtype=np.float64)), kw["lo"], kw["hi"])
            r = H.eval_encrypted(ctx, s, H.Ciphertext(kw["x"], kw["lx"]))
            out, levels = r.slots(), [r.level()]
        elif api == "newton_refine":
            r = H.newton_refine(ctx, H.Ciphertext(kw["x"], kw["lx"]), H.Ciphertext(kw["y0"], kw["ly"]), kw["n"],
                                kw["iters"], kw["n_valid"])
            out, levels = r.slots(), [r.level()]
        elif api == "invroot":
            x = H.Ciphertext(kw["x"], kw["lx"])
            cfg = cfg_of(kw.get("cfg"))
            w = kw["which"]
            if w == 0:
                r = H.crypto_invsqrt(ctx, x, kw["S"], cfg, kw["n_valid"])
            elif w == 1:
                r = H.crypto_inv(ctx, x, kw["S"], cfg, kw["n_valid"])
            elif w == 2:
                r = H.baseline_invsqrt(ctx, x, kw["S"], cfg.newton_iters, kw["n_valid"])
            else:
                r = H.crypto_sqrt(ctx, x, kw["S"], cfg.cheb_degree, kw["n_valid"])
            out, levels = r.slots(), [r.level()]
        elif api == "crypto_sign":
            sc = H.SignConfig(H.SignMode(kw["mode"]), kw["folds"], [list(p) for p in kw["polys"]])
            r = H.crypto_sign(ctx, H.Ciphertext(kw["x"], kw["lx"]), sc)
            out, levels = r.slots(), [r.level()]
        elif api == "stat":
            which, B = kw["which"], kw["B"]
            cfg = cfg_of(kw.get("cfg"))
            col = H.encode_column(ctx, kw["x"], "x")
            if which == 0:
                r = H.mean_scaled(ctx, col, B)
            elif which == 1:
                r = H.variance_scaled(ctx, col, B)
            elif which == 2:
                r = H.variance_to_scale(ctx, col, B)
            elif which == 3:
                m = H.moments(ctx, col, B)
                out = np.concatenate([m.ct_mu.slots(), m.ct_var.slots()])
                levels = [m.ct_mu.level(), m.ct_var.level()]
                r = None
            elif which == 4:
                z = H.znorm(ctx, col, B, cfg)
                out = H.decode_column(ctx, z)
                levels = [z.chunks[0].level() if z.chunks else 0]
                r = None
            elif which == 5:
                r = H.kurtosis(ctx, col, B, cfg)
            elif which == 6:
                r = H.skewness(ctx, col, B, cfg)
            elif which == 7:
                r = H.coeff_variation(ctx, col, B, H.SignConfig(), cfg)
            else:
                r = H.pearson(ctx, col, H.encode_column(ctx, kw["y"], "y"), B, cfg)
            if r is not None:
                out, levels = r.slots(), [r.level()]
        else:
            raise ValueError(api)
        rc = 0
    except H.error as e:
        rc = _code(e)
    m = ctx.meter().as_tuple()
    return rc, np.asarray(out, dtype=np.float64), tuple(levels), m
