"""Scales other than 2^-40 on the fused path (the magic-constant rounding in the
Chebyshev core is exact only below 2^51 grid units, so its enabling bound must shrink with
scale_bits; very large scales must leave the grid-unit kernels).  znorm and coeff_variation
(whose crypto_sqrt has leaves of ~141 real units at B = 100) at scale_bits 30, 45, 50 and 420
are bit-exact against the C oracle and, where it was built, the compiled reference."""
import numpy as np
import pytest

from oracle_abi import Params, ST_CV, ST_ZNORM, bits, oracle, reference


def _check(which, sb, x, B):
    from paper_2508_12093_b200 import hestat as H
    S = 4096
    ctx = H.EvalContext(H.CkksParams(slot_count=S, scale_bits=sb))
    col = H.encode_column(ctx, x)
    if which == ST_ZNORM:
        got = H.decode_column(ctx, H.znorm(ctx, col, B))
    else:
        got = ctx.decrypt(H.coeff_variation(ctx, col, B), 1)
    for lib in (oracle(), reference()):
        if lib is None:
            continue
        ref = lib.stat(Params(slot_count=S, scale_bits=sb), which, x, B)
        assert ref.rc == 0
        assert np.array_equal(bits(got), bits(ref.out[: got.size])), (lib.path, sb)
        assert ctx.meter().as_tuple() == ref.meter


@pytest.mark.gpu
@pytest.mark.parametrize("sb", [30, 45, 50, 420])
def test_znorm_scale_bits(sb):
    from paper_2508_12093_b200 import hestat as H
    _check(ST_ZNORM, sb, 50.0 + 10.0 * (H.synthetic_uniform(3, 4000, 0.0, 1.0) - 0.5), 100.0)


@pytest.mark.gpu
@pytest.mark.parametrize("sb", [30, 45, 50, 420])
def test_coeff_variation_scale_bits(sb):
    from paper_2508_12093_b200 import hestat as H
    _check(ST_CV, sb, H.synthetic_uniform(1004, 4000, 0.0, 20.0) + 30.0, 100.0)
