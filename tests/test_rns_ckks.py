"""GPU: Tier-R encryption / decryption and the decrypted semantics of every
Tier-R op (ckks.hpp op semantics realised over RNS-CKKS):

  * encrypt_coeffs / decrypt_coeffs limb-exact vs the RNS oracle;
  * decrypt(encrypt(x)) = x, add / sub / add_const / mul_const;
  * HMult+relin+rescale: decrypt = x*y at scale D^2/q_l (two levels deep too);
  * rotate(k): decrypt = left rotation by k (ckks.hpp:193-202);
at the CKKS precision of scale 2^40 (errors ~1e-9..1e-7 absolute).
"""
import numpy as np
import pytest

from rns_abi import RnsOracle, Spec

pytestmark = pytest.mark.gpu

O = RnsOracle()
SP = Spec(logN=12, L=5, K=2, dnum=3, seed=17)
DELTA = 2.0 ** 40


def _ctx(s):
    from paper_2508_12093_b200.rns import RnsContext, RnsSpec
    return RnsContext(RnsSpec(s.logN, s.L, s.K, s.dnum, s.logq0, s.logq, s.logp, seed=s.seed, h=s.h))


@pytest.fixture(scope="module")
def ctx():
    return _ctx(SP)


def _x(seed, n, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, n)


@pytest.mark.parametrize("level", [5, 2, 0])
def test_encrypt_limb_exact(ctx, level):
    rng = np.random.default_rng(level)
    m = rng.integers(-(2 ** 45), 2 ** 45, SP.N)
    ct = ctx.encrypt_coeffs(level, m, tag=3 + level)
    assert np.array_equal(ct.download(), O.encrypt_coeffs(SP, level, m, 3 + level))
    d = ctx.decrypt_coeffs(level, ct)
    assert np.array_equal(d, O.decrypt_coeffs(SP, level, ct.download()))
    assert np.max(np.abs(d - m)) <= 21


def test_encrypt_decrypt_values(ctx):
    S = SP.N // 2
    x = _x(1, S, -100, 100)
    ct = ctx.encrypt(SP.L, x, DELTA, tag=1)
    assert np.max(np.abs(ctx.decrypt(SP.L, ct, DELTA) - x)) < 1e-7
    # partial vectors are zero padded (ckks.hpp:97-104)
    ct2 = ctx.encrypt(SP.L, x[:100], DELTA, tag=2)
    y = ctx.decrypt(SP.L, ct2, DELTA)
    assert np.max(np.abs(y[:100] - x[:100])) < 1e-7 and np.max(np.abs(y[100:])) < 1e-7


def test_add_sub_const(ctx):
    S = SP.N // 2
    x, y = _x(2, S), _x(3, S)
    a, b = ctx.encrypt(SP.L, x, DELTA, 10), ctx.encrypt(SP.L, y, DELTA, 11)
    assert np.max(np.abs(ctx.decrypt(SP.L, ctx.add(SP.L, a, b), DELTA) - (x + y))) < 1e-7
    assert np.max(np.abs(ctx.decrypt(SP.L, ctx.add(SP.L, a, b, sub=True), DELTA) - (x - y))) < 1e-7
    c = ctx.add_const(SP.L, a, int(round(-0.75 * DELTA)))
    assert np.max(np.abs(ctx.decrypt(SP.L, c, DELTA) - (x - 0.75))) < 1e-7
    m = ctx.mul_const(SP.L, a, -3)
    assert np.max(np.abs(ctx.decrypt(SP.L, m, DELTA) - (-3 * x))) < 1e-7


def test_hmult_decrypts_to_product(ctx):
    S = SP.N // 2
    primes = [int(p) for p in ctx.primes()]
    x, y, z = _x(4, S), _x(5, S), _x(6, S)
    l = SP.L
    a, b, c = (ctx.encrypt(l, v, DELTA, 20 + i) for i, v in enumerate((x, y, z)))
    ab = ctx.mul_relin_rescale(l, a, b)
    s1 = DELTA * DELTA / primes[l]
    assert np.max(np.abs(ctx.decrypt(l - 1, ab, s1) - x * y)) < 1e-6
    # two levels deep: (x*y) * z with z brought to the same scale and level
    c1 = ctx.rescale(l, ctx.mul_const(l, c, int(round(s1 * primes[l] / DELTA))))
    abc = ctx.mul_relin_rescale(l - 1, ab, c1)
    s2 = s1 * s1 / primes[l - 1]
    assert np.max(np.abs(ctx.decrypt(l - 2, abc, s2) - x * y * z)) < 1e-5


@pytest.mark.parametrize("k", [1, 5, -3, 1024])
def test_rotate_decrypts_to_left_rotation(ctx, k):
    S = SP.N // 2
    x = _x(7, S)
    a = ctx.encrypt(SP.L, x, DELTA, 30)
    r = ctx.rotate(SP.L, k, a)
    assert np.max(np.abs(ctx.decrypt(SP.L, r, DELTA) - np.roll(x, -k))) < 1e-6


def test_sum_all_slots_by_rotations(ctx):
    """The reference's sum_all_slots (ckks.hpp:218-230): log2 S rotate-and-add steps."""
    S = SP.N // 2
    x = _x(8, S)
    acc = ctx.encrypt(SP.L, x, DELTA, 40)
    step = 1
    while step < S:
        acc = ctx.add(SP.L, acc, ctx.rotate(SP.L, step, acc))
        step <<= 1
    out = ctx.decrypt(SP.L, acc, DELTA)
    assert np.max(np.abs(out - x.sum())) < 1e-5


def test_full_size_round_trip():
    s = Spec(logN=16, L=24, K=9, dnum=3, seed=2)
    c = _ctx(s)
    S = s.N // 2
    x, y = _x(9, S, 0, 100), _x(10, S, -1, 1)
    a, b = c.encrypt(s.L, x, DELTA, 1), c.encrypt(s.L, y, DELTA, 2)
    assert np.max(np.abs(c.decrypt(s.L, a, DELTA) - x)) < 1e-6
    p = c.mul_relin_rescale(s.L, a, b)
    s1 = DELTA * DELTA / int(c.primes()[s.L])
    assert np.max(np.abs(c.decrypt(s.L - 1, p, s1) - x * y)) < 1e-5
    r = c.rotate(s.L, 7, a)
    assert np.max(np.abs(c.decrypt(s.L, r, DELTA) - np.roll(x, -7))) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("logN", [4, 10, 12, 16])
def test_device_codec_bit_identical_to_host(logN):
    """codec_gpu.cu (used by RNS-backed EvalContexts) vs rns_codec.cpp: same FFT, same roundings."""
    from paper_2508_12093_b200 import rns as R
    rng = np.random.default_rng(logN)
    S = 1 << (logN - 1)
    for n, scale in ((S, 2.0 ** 40), (S // 2 + 1, 2.0 ** 30), (1, 2.0 ** 20)):
        z = rng.uniform(-3.0, 3.0, n)
        host = R.encode(logN, z, scale)  # int64 (no signed zero); the device gives integral doubles
        dev = R.encode_gpu(logN, z, scale)
        assert np.array_equal(host.astype(np.float64), dev) and np.array_equal(np.rint(dev), dev), (logN, n)
        back_h = R.decode(logN, host, scale, n)
        back_d = R.decode_gpu(logN, dev, scale, n)
        assert np.array_equal(back_h.view(np.int64), back_d.view(np.int64)), (logN, n)
        assert np.max(np.abs(back_d - z)) < (1 << logN) / scale
