"""Pins of the CPU oracle (oracle/q4_oracle.c) against things other than
itself: IEEE/numpy conversions exhaustively, hand-derived closed forms
(tests/golden/), exact rational brute force, and invariants.

None of these tests re-types the oracle's formulas in the same form: code
extraction is done with Python integer loops, dequant with numpy's float32
multiply + float16 cast, sums with fractions.Fraction or integer numpy.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- helpers
def pack_py(codes_rows):
    """Independent packer: list of code lists -> uint32 words (pure Python)."""
    out = []
    for row in codes_rows:
        words = []
        for w in range(len(row) // 8):
            v = 0
            for t in range(8):
                v |= (int(row[8 * w + t]) & 0xF) << (4 * t)
            words.append(v)
        out.append(words)
    return np.array(out, dtype=np.uint32)


def codes_py(packed, K):
    """Independent unpacker with Python ints: [N][K] codes."""
    N = packed.shape[0]
    out = np.zeros((N, K), dtype=np.int64)
    for j in range(N):
        for k in range(K):
            word = int(packed[j, k // 8])
            out[j, k] = (word >> (4 * (k % 8))) & 15
    return out


def numpy_W(packed, scales, K):
    """W via numpy: float32 product (exact: <=15 significant bits) then one
    float16 cast (numpy rounds to nearest even).  [N][K] float16."""
    q = codes_py(packed, K)
    s = scales.view(np.float16).astype(np.float32)
    s_full = np.repeat(s, 32, axis=1)
    with np.errstate(invalid="ignore", over="ignore"):
        return (np.float32(1.0) * (q - 7).astype(np.float32) * s_full).astype(np.float16)


def f16(bits):
    return np.asarray(bits, dtype=np.uint16).view(np.float16)


def same_bits_or_both_nan(a_bits, b_bits):
    a = np.asarray(a_bits, dtype=np.uint16)
    b = np.asarray(b_bits, dtype=np.uint16)
    a_nan = np.isnan(a.view(np.float16))
    b_nan = np.isnan(b.view(np.float16))
    return np.array_equal(a_nan, b_nan) and np.array_equal(a[~a_nan], b[~b_nan])


# ---------------------------------------------------------------- dequant
def test_dequant_exhaustive_all_codes_all_scale_bits():
    """All 16 codes x all 65536 fp16 scale bit patterns (1,048,576 pairs):
    oracle == numpy float32 multiply + float16 cast, bit for bit (NaN by
    class).  SURVEY §8(c) 'Dequant, exhaustively'."""
    N, K = 65536, 32
    codes = np.tile(np.concatenate([np.arange(16), np.arange(16)]), (N, 1))
    packed = inputs.pack_codes(codes.astype(np.uint8))
    scales = np.arange(N, dtype=np.uint32).astype(np.uint16).reshape(N, 1)
    got = oracle.dequant(packed, scales, K, N)
    s = scales.view(np.float16).astype(np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        want = ((codes.astype(np.float32) - np.float32(7)) * s).astype(np.float16)
    assert same_bits_or_both_nan(got, want.view(np.uint16))


def _golden_dequant():
    rows = []
    with open(os.path.join(GOLDEN, "dequant_spot.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            c, s, e = line.split()
            rows.append((int(c), int(s, 16), e))
    return rows


@pytest.mark.parametrize("code,scale,expected", _golden_dequant())
def test_dequant_golden_spot_values(code, scale, expected):
    row = [7] * 32
    row[5] = code                      # element k=5 of group 0
    packed = pack_py([row])
    scales = np.array([[scale]], dtype=np.uint16)
    w = oracle.dequant(packed, scales, 32, 1)[0, 5]
    if expected == "nan":
        assert np.isnan(f16(w))
    else:
        assert int(w) == int(expected, 16), f"{int(w):#06x} != {expected}"


def test_nibble_order_words():
    """0x76543210 -> codes 0..7 -> W = (-7..0)*s; 0xFEDCBA98 -> (1..8)*s."""
    packed = np.array([[0x76543210, 0xFEDCBA98, 0x76543210, 0xFEDCBA98]], dtype=np.uint32)
    scales = np.array([[0x3800]], dtype=np.uint16)  # s = 0.5
    w = f16(oracle.dequant(packed, scales, 32, 1)[0]).astype(np.float64)
    want = np.array([(t - 7) * 0.5 for t in range(16)] * 2)
    assert np.array_equal(w, want)


def test_dequant_groups_are_32_consecutive_k():
    """Scale g applies to k in [32g, 32g+32) and to no other k (reading 2)."""
    K, N = 128, 3
    packed = pack_py([[15] * K] * N)            # W = 8*s everywhere
    sc = np.array([[0x3c00, 0x4000, 0x4400, 0x4800]] * N, dtype=np.uint16)  # 1,2,4,8
    w = f16(oracle.dequant(packed, sc, K, N)).astype(np.float64)
    for g, s in enumerate([1, 2, 4, 8]):
        assert np.all(w[:, 32 * g:32 * g + 32] == 8 * s)


def test_dequant_random_matches_numpy():
    K, N = 256, 64
    packed, scales = inputs.stress_weights(11, K, N)
    got = oracle.dequant(packed, scales, K, N)
    assert np.array_equal(got, numpy_W(packed, scales, K).view(np.uint16))


# ---------------------------------------------------------------- round
def test_round_f16_against_numpy_and_closed_forms():
    g = np.random.default_rng(3)
    r = np.concatenate([
        g.standard_normal(20000) * 10.0 ** g.integers(-9, 6, 20000),
        np.array([65504.0, 65519.99, 65520.0, -65520.0, 2.0 ** -25, 2.0 ** -24 * 1.5,
                  2.0 ** -26, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 0.0, -0.0,
                  1.0 + 2.0 ** -11 + 2.0 ** -40]),
    ])
    got = oracle.round_f16(r)
    with np.errstate(over="ignore"):
        want = r.astype(np.float16).view(np.uint16)
    assert np.array_equal(got, want)
    # closed forms: max finite stays, 65520 is the overflow tie -> inf,
    # 1+2^-11 ties to even (1.0), 1+3*2^-11 ties to even (1+2^-9)
    assert got[-12] == 0x7BFF and got[-10] == 0x7C00 and got[-9] == 0xFC00
    assert got[-5] == 0x3C00 and got[-4] == 0x3C02
    assert got[-3] == 0x0000 and got[-2] == 0x8000
    assert got[-1] == 0x3C01  # just above the tie -> rounds up


def test_f16_to_f64_exhaustive():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    got = oracle.f16_to_f64(bits)
    want = bits.view(np.float16).astype(np.float64)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint64), want[~nan].view(np.uint64))


# ---------------------------------------------------------------- matmul
def exact_r(x_bits, packed, scales, K):
    """Exact rational r via fractions.Fraction, W from numpy_W."""
    W = numpy_W(packed, scales, K).astype(np.float64)   # [N][K], exact fp16 values
    X = f16(x_bits).astype(np.float64)
    n, N = X.shape[0], W.shape[0]
    out = [[None] * N for _ in range(n)]
    abs_sum = np.zeros((n, N))
    for i in range(n):
        for j in range(N):
            acc = Fraction(0)
            a = 0.0
            for k in range(K):
                term = Fraction(float(X[i, k])) * Fraction(float(W[j, k]))
                acc += term
                a += abs(float(term))
            out[i][j] = acc
            abs_sum[i, j] = a
    return out, abs_sum


@pytest.mark.parametrize("K", [32, 64])
@pytest.mark.parametrize("N", [1, 2, 3, 8])
@pytest.mark.parametrize("n", [1, 2, 3])
def test_matmul_vs_exact_rational(K, N, n):
    packed, scales = inputs.stress_weights(100 + K + N, K, N)
    x = inputs.activations(7 + n, n, K, "uniform")
    r = oracle.matmul_f64(x, packed, scales, K, N)
    exact, abs_sum = exact_r(x, packed, scales, K)
    for i in range(n):
        for j in range(N):
            err = abs(Fraction(float(r[i, j])) - exact[i][j])
            bound = K * 2.0 ** -53 * abs_sum[i, j] * 1.01
            assert float(err) <= bound


def test_matmul_exact_on_small_dyadics():
    """x in {-1,-0.5,0,0.5,1}, scales powers of two: every partial sum is a
    short dyadic, so fp64 must equal the exact rational result."""
    K, N, n = 64, 8, 3
    g = np.random.default_rng(5)
    codes = g.integers(0, 16, size=(N, K))
    packed = pack_py(codes.tolist())
    scales = f16(np.zeros((N, K // 32))).copy()
    scales = (2.0 ** g.integers(-6, 3, size=(N, K // 32))).astype(np.float16).view(np.uint16)
    x = g.choice([-1.0, -0.5, 0.0, 0.5, 1.0], size=(n, K)).astype(np.float16).view(np.uint16)
    r = oracle.matmul_f64(x, packed, scales, K, N)
    exact, _ = exact_r(x, packed, scales, K)
    for i in range(n):
        for j in range(N):
            assert Fraction(float(r[i, j])) == exact[i][j]


def test_matmul_golden_closed_form():
    # tests/golden/matmul_closed_form.txt
    K = 32
    packed = pack_py([[15] * 32, list(range(16)) * 2])
    scales = np.array([[0x3400], [0x3800]], dtype=np.uint16)
    x = np.full((1, K), 0x3C00, dtype=np.uint16)
    r = oracle.matmul_f64(x, packed, scales, K, 2)
    assert r[0, 0] == 64.0 and r[0, 1] == 8.0


@pytest.mark.parametrize("case", ["codes7", "scales0", "x0"])
def test_zero_invariants(case):
    K, N, n = 256, 16, 4
    packed, scales = inputs.stress_weights(21, K, N)
    x = inputs.activations(22, n, K)
    if case == "codes7":
        packed = np.full_like(packed, 0x77777777)
    elif case == "scales0":
        scales = np.zeros_like(scales)
    else:
        x = np.zeros_like(x)
    r = oracle.matmul_f64(x, packed, scales, K, N)
    assert np.all(r == 0.0)


def test_identity_scale_integer_exact():
    """scales = 1.0, x in {-1,0,1}: r = sum (q-7) x computed in integers."""
    K, N, n = 512, 32, 5
    g = np.random.default_rng(9)
    packed = g.integers(0, 2**32, size=(N, K // 8), dtype=np.uint64).astype(np.uint32)
    scales = np.full((N, K // 32), 0x3C00, dtype=np.uint16)
    xi = g.integers(-1, 2, size=(n, K))
    x = xi.astype(np.float16).view(np.uint16)
    r = oracle.matmul_f64(x, packed, scales, K, N)
    q = codes_py(packed, K)
    want = xi @ (q - 7).T
    assert np.array_equal(r, want.astype(np.float64))


def test_one_hot_extracts_W():
    K, N = 128, 24
    packed, scales = inputs.stress_weights(31, K, N)
    ks = [0, 1, 31, 32, 77, 127]
    x = np.zeros((len(ks), K), dtype=np.uint16)
    for i, k in enumerate(ks):
        x[i, k] = 0x3C00
    r = oracle.matmul_f64(x, packed, scales, K, N)
    W = numpy_W(packed, scales, K).astype(np.float64)
    for i, k in enumerate(ks):
        assert np.array_equal(r[i], W[:, k])


def test_rows_independent_prefix_and_cols_and_threads():
    K, N, n = 256, 48, 9
    packed, scales = inputs.realistic_weights(41, K, N)
    x = inputs.activations(42, n, K)
    full = oracle.matmul_f64(x, packed, scales, K, N, nthreads=4)
    one = oracle.matmul_f64(x, packed, scales, K, N, nthreads=1)
    assert np.array_equal(full.view(np.uint64), one.view(np.uint64))
    for m in (1, 4, 9):
        part = oracle.matmul_f64(x[:m], packed, scales, K, N)
        assert np.array_equal(part, full[:m])
    cols = [0, 5, 47, 5]
    rc = oracle.matmul_cols_f64(x, packed, scales, K, cols)
    assert np.array_equal(rc, full[:, cols])


def test_realistic_generator_matches_recipe():
    """The test-data quantiser emits codes 0..14 with max |q-7| == 7 in every
    group whose scale is nonzero (recipe)."""
    K, N = 256, 16
    packed, scales = inputs.realistic_weights(3, K, N)
    q = codes_py(packed, K).reshape(N, K // 32, 32)
    assert q.max() <= 14
    assert np.all(np.abs(q - 7).max(axis=2)[f16(scales) != 0] == 7)
