"""CPU: the C-ABI library loads, exports every symbol include/hestat_gpu.h
declares, and its host-side helpers (fit, Clenshaw, data generators, plain
statistics — host code in the reference too) agree with the oracle.  No call
here touches a GPU."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from oracle_abi import ROOT, FIT_EXP, FIT_INVSQRT_SHIFTED, FIT_SQRT_SHIFTED, bits, oracle

HEADERS = [os.path.join(ROOT, "include", h) for h in ("hestat_gpu.h", "hestat_rns.h")]
LIB = os.path.join(ROOT, "paper_2508_12093_b200", "libhestat_gpu.so")


def declared():
    txt = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", txt)) - {"hs_target_fn"})


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared()) >= 60


def test_python_binding_covers_header():
    from paper_2508_12093_b200 import _abi
    assert set(declared()) == set(_abi.symbols())


def test_sm100a_cubin_present():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("kind,S,deg", [(FIT_INVSQRT_SHIFTED, 100.0, 511), (FIT_INVSQRT_SHIFTED, 1.0, 15),
                                        (FIT_SQRT_SHIFTED, 400.0, 511), (FIT_INVSQRT_SHIFTED, 2.0, 0)])
def test_fit_matches_oracle(kind, S, deg):
    from paper_2508_12093_b200 import hestat as H
    s = H.fit_scaled(H.ScaledTargetKind(kind), S, deg)
    rc, ref = oracle().fit(kind, S, deg)
    assert rc == 0 and np.array_equal(bits(np.asarray(s.coeffs)), bits(ref))
    s2 = H.fit(lambda t: H.scaled_target(H.ScaledTargetKind(kind), S, t), deg)
    assert np.array_equal(bits(np.asarray(s2.coeffs)), bits(ref))


def test_fit_callback_and_errors():
    from paper_2508_12093_b200 import hestat as H
    s = H.fit(math.exp, 63)
    rc, ref = oracle().fit(FIT_EXP, 1, 63)
    assert np.array_equal(bits(np.asarray(s.coeffs)), bits(ref))
    with pytest.raises(H.non_finite_target):
        H.fit(math.sqrt if False else (lambda x: float("nan")), 8)
    with pytest.raises(H.error):
        H.fit(math.exp, -1)
    ex = []
    v = H.eval_plain(H.ChebyshevSeries([0.0, 1.0]), 1.5, ex)
    assert v == 1.5 and ex == [True]
    assert H.cheb_eval_depth(511) == 9 and H.cheb_eval_depth(0) == 0


def test_data_helpers_match_oracle():
    from paper_2508_12093_b200 import hestat as H
    o = oracle()
    assert np.array_equal(bits(H.synthetic_uniform(42, 1000, 0.0, 100.0)), bits(o.synthetic_uniform(42, 1000, 0.0, 100.0)))
    assert np.array_equal(bits(H.two_subrange_grid(32768, 0.001, 100.0)), bits(o.two_subrange_grid(32768, 0.001, 100.0)))
    x = o.synthetic_uniform(3, 999, 0.5, 20.0)
    y = o.synthetic_uniform(4, 999, 0.5, 20.0)
    for which, f in [(0, H.plain.mean), (1, H.plain.variance), (2, H.plain.skewness), (3, H.plain.kurtosis_ratio),
                     (4, H.plain.coeff_variation)]:
        assert f(x) == o.plain(which, x)[1]
    assert H.plain.pearson(x, y) == o.plain(5, x, y)[1]
    assert np.array_equal(bits(H.plain.znorm(x)), bits(o.plain(6, x)[1]))
    with pytest.raises(H.zero_reference):
        H.mre([1.0], [0.0])
    with pytest.raises(H.empty_column):
        H.plain.mean([])
