"""Pins of the fused-neighbour oracle (oracle/fused.py) against values the
mathematics fixes -- closed forms worked by hand, invariants and special
cases -- so a dropped term, a wrong rounding point or a swapped pair fails
here before any GPU comparison trusts it."""
import math

import numpy as np

import oracle
from oracle import fused as fo


def f16bits(vals):
    return np.asarray(vals, dtype=np.float64).astype(np.float16).view(np.uint16)


def f64(bits):
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


def test_rmsnorm_worked_example():
    # x = [3, 4]: mean x^2 = 12.5, r = 1/sqrt(12.5).  By hand:
    #   3 r = 0.84852813...; fp16 spacing in [0.5, 1) is 2^-11: 1737.79 ulps -> 1738 * 2^-11 = 0.8486328125
    #   4 r = 1.13137085...; spacing in [1, 2) is 2^-10: 1158.52 ulps -> 1159 * 2^-10 = 1.1318359375
    # gamma = [1, 0.5] halves the second exactly.
    xn = fo.rmsnorm_x(f16bits([[3.0, 4.0]]), f16bits([1.0, 0.5]), 0.0)
    assert f64(xn).tolist() == [[0.8486328125, 0.56591796875]]


def test_rmsnorm_constant_row_is_unit():
    for c in (0.001, -3.5, 1000.0):
        xn = fo.rmsnorm_x(f16bits([[c] * 64]), f16bits([1.0] * 64), 0.0)
        assert np.all(f64(xn) == math.copysign(1.0, c))


def test_rmsnorm_scale_invariance_and_gamma():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 256)).astype(np.float16)
    g = rng.uniform(0.5, 2.0, 256).astype(np.float16)
    a = fo.rmsnorm_x(x.view(np.uint16), g.view(np.uint16), 0.0)
    b = fo.rmsnorm_x((x * np.float16(8.0)).view(np.uint16), g.view(np.uint16), 0.0)   # exact power of two
    assert np.array_equal(a, b)
    # gamma = 1: the RMS of the output row is 1 up to fp16 rounding
    one = fo.rmsnorm_x(x.view(np.uint16), f16bits([1.0] * 256), 0.0)
    rms = np.sqrt(np.mean(f64(one) ** 2, axis=1))
    assert np.all(np.abs(rms - 1.0) < 1e-3)


def test_rmsnorm_eps():
    # eps dominates a tiny row: r = 1/sqrt(mean + eps) ~ 1/sqrt(eps)
    x = f16bits([[1e-4] * 32])
    xn = fo.rmsnorm_x(x, f16bits([1.0] * 32), 1.0)
    assert np.all(np.abs(f64(xn) - 1e-4 / math.sqrt(1.0 + 1e-8)) < 1e-7)


def test_silu_closed_forms():
    assert fo.silu(np.array([0.0]))[0] == 0.0
    assert abs(fo.silu(np.array([1.0]))[0] - 0.7310585786300049) < 1e-15     # sigmoid(1) = e / (1 + e)
    assert abs(fo.silu(np.array([-1.0]))[0] + 0.2689414213699951) < 1e-15
    assert abs(fo.silu(np.array([30.0]))[0] - 30.0) < 1e-10
    assert fo.silu(np.array([-1000.0]))[0] == 0.0


def test_silu_mul_pairs_and_rounding_point():
    # r over interleaved rows: (gate, up) = (1, 2) and (-1, 3); gate/up are
    # rounded to fp16 before the SiLU (the unfused matmul stores fp16)
    r = np.array([[1.0, 2.0, -1.0, 3.0]])
    y = fo.silu_mul(r)
    assert np.allclose(y, [[0.7310585786300049 * 2.0, -0.2689414213699951 * 3.0]], rtol=0, atol=1e-15)
    r2 = np.array([[1.0 + 2.0 ** -12, 1.0]])              # below half an fp16 ulp: rounds to 1.0
    assert fo.silu_mul(r2)[0, 0] == fo.silu(np.array([1.0]))[0]


def test_residual_with_zero_weights_is_identity():
    # codes 7 -> W = 0 exactly -> the matmul is +-0 and the residual passes through
    K, N = 64, 8
    packed = np.full((N, K // 8), 0x77777777, dtype=np.uint32)
    scales = f16bits(np.ones((N, K // 32)))
    x = f16bits(np.linspace(-1, 1, K)[None, :])
    r = oracle.matmul_f64(x, packed, scales, K, N)
    res = f16bits(np.arange(N)[None, :] * 0.25)
    assert np.array_equal(fo.residual(r, res), f64(res))


def test_interleave_rows():
    a = np.arange(6).reshape(3, 2)
    b = -np.arange(6).reshape(3, 2)
    out = fo.interleave_rows(a, b)
    assert out.tolist() == [[0, 1], [0, -1], [2, 3], [-2, -3], [4, 5], [-4, -5]]


def test_residual_rounds_v_to_fp16_first():
    """Reading 18: the residual adds the fp16 OUTPUT of the matmul (the
    unfused chain stores it): r = 1 + 2^-12 is below half an fp16 ulp of 1
    (2^-11), so it contributes exactly 1.0; r = 1 + 3 * 2^-12 rounds up to
    1 + 2^-10; ties go to even (1 + 2^-11 -> 1.0, 1 + 3 * 2^-11 -> 1 + 2^-9)."""
    res = f16bits(np.array([[0.5, 0.5, 0.5, 0.5]]))
    r = np.array([[1.0 + 2.0 ** -12, 1.0 + 3 * 2.0 ** -12, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11]])
    y = fo.residual(r, res)
    assert y.tolist() == [[1.5, 1.5 + 2.0 ** -10, 1.5, 1.5 + 2.0 ** -9]]
    # the fp16 bits path gives the same value as the float path
    vb = f16bits(np.array([[1.0, 1.0 + 2.0 ** -10]]))
    assert fo.residual(vb, res[:, :2], v_is_bits=True).tolist() == [[1.5, 1.5 + 2.0 ** -10]]
    # overflow of v itself: fp16(70000) = inf, not 70000
    assert np.isinf(fo.residual(np.array([[70000.0]]), f16bits(np.array([[-1.0]])))[0, 0])
