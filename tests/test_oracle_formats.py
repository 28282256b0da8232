"""Pins of oracle/formats.py (the format variants of SURVEY §8(f) F3) against
the C oracle's dequant of the native format and hand-worked values."""
import numpy as np
import pytest

import oracle
from oracle import formats as fm
from paper_2311_02103_b200 import inputs


def kn_pack(q):
    """codes uint8 [N][K] -> KN words [K/8][N], written as plain loops (independent
    of formats.codes): word (k8, j) = sum_i q[j][8 k8 + i] << 4 i."""
    N, K = q.shape
    out = np.zeros((K // 8, N), dtype=np.uint32)
    for k8 in range(K // 8):
        for i in range(8):
            out[k8] |= q[:, 8 * k8 + i].astype(np.uint32) << np.uint32(4 * i)
    return out


def test_hand_worked_kn_word():
    # column 1, k = 0..7 hold codes 0..7 (word 0x76543210); scale 0.5 for the
    # first 64-group of column 1, 2.0 for column 0
    K, N, G = 64, 2, 64
    packed = np.full((K // 8, N), 0x77777777, dtype=np.uint32)
    packed[0, 1] = 0x76543210
    scales = np.array([[0x4000, 0x3800]], dtype=np.uint16)        # [K/G][N]: 2.0, 0.5
    W = fm.dequant(packed, scales, K, N, "kn", G).view(np.float16).astype(np.float64)
    assert W[1, :8].tolist() == [(q - 7) * 0.5 for q in range(8)]
    assert np.all(W[1, 8:] == 0) and np.all(W[0] == 0)


@pytest.mark.parametrize("layout", fm.LAYOUTS)
@pytest.mark.parametrize("group", fm.GROUPS)
def test_format_matches_native_oracle(layout, group):
    """A weight stored in (layout, G) dequantizes, bit for bit, to the C
    oracle's dequant of its native conversion, and to_native agrees with an
    independent construction of the native format."""
    K, N = 256, 24
    rng = np.random.default_rng(group + len(layout))
    q = rng.integers(0, 16, size=(N, K), dtype=np.uint8)
    sg = rng.uniform(2.0 ** -10, 2.0 ** -3, size=(N, K // group)).astype(np.float16).view(np.uint16)
    if layout == "nk":
        src_p, src_s = inputs.pack_codes(q), sg
    else:
        src_p, src_s = kn_pack(q), np.ascontiguousarray(sg.T)
    W = fm.dequant(src_p, src_s, K, N, layout, group)
    nat_p, nat_s = fm.to_native(src_p, src_s, K, N, layout, group)
    assert np.array_equal(nat_p, inputs.pack_codes(q))
    assert np.array_equal(nat_s, np.repeat(sg, group // 32, axis=1))
    assert np.array_equal(W, oracle.dequant(nat_p, nat_s, K, N))


# ---- 3-bit ("nk3", reading 20) -------------------------------------
# Hand-worked group: codes c_i = i mod 8.  Word 0 = codes 0..7 in bits 0..23
# (0b111_110_101_100_011_010_001_000 = 0xFAC688), code 8 = 0 in bits 24..26,
# code 9 = 1 sets bit 27, code 10 = 2 = 0b010 puts its middle bit at bit 31
# (bits 30..32 straddle words 0 and 1): word 0 = 0x88FAC688; the pattern
# repeats every 8 codes = 24 bits, giving words 1 and 2 below.
Q3_GOLDEN_WORDS = [0x88FAC688, 0xC688FAC6, 0xFAC688FA]


def test_q3_hand_worked_words():
    q = fm.codes3(np.array([Q3_GOLDEN_WORDS], dtype=np.uint32), 32, 1)
    assert q[0].tolist() == [i % 8 for i in range(32)]


def test_q3_zero_point_and_word_boundaries():
    """All codes 3 -> W == 0 exactly; a single code 7 at every position --
    including 10 and 21, which straddle the words -- gives exactly one weight
    4 * s and zeros elsewhere."""
    # all-3 group: 0b011 repeated = bits 0,1, 3,4, ... of the 96-bit triple
    bits = sum(3 << (3 * i) for i in range(32))
    w3 = [(bits >> (32 * k)) & 0xFFFFFFFF for k in range(3)]
    s = np.array([[0x2E00]], dtype=np.uint16)                      # 0.09375
    W = fm.dequant3(np.array([w3], dtype=np.uint32), s, 32, 1, 32)
    assert np.all(W == 0)
    for pos in range(32):
        b = bits & ~(7 << (3 * pos)) | (7 << (3 * pos))
        w = [(b >> (32 * k)) & 0xFFFFFFFF for k in range(3)]
        W = fm.dequant3(np.array([w], dtype=np.uint32), s, 32, 1, 32)
        want = np.zeros(32, dtype=np.uint16)
        want[pos] = 0x3600                                         # 4 * 0.09375 = 0.375
        assert np.array_equal(W[0], want), pos


@pytest.mark.parametrize("group", [32, 64, 128])
def test_q3_native_form_dequantizes_identically(group):
    """to_native(q3) read by the (separately pinned) q4 definitions gives the
    same W as the q3 definition, for random words (every 96-bit pattern is a
    valid code triple) and every code value."""
    K, N = 256, 7
    rng = np.random.default_rng(group)
    p3 = rng.integers(0, 2 ** 32, size=(N, K // 32 * 3), dtype=np.uint64).astype(np.uint32)
    s = rng.uniform(2.0 ** -10, 2.0 ** -4, size=(N, K // group)).astype(np.float16).view(np.uint16)
    W3 = fm.dequant3(p3, s, K, N, group)
    pk, sc = fm.to_native(p3, s, K, N, "nk3", group)
    assert np.array_equal(oracle.dequant(pk, sc, K, N), W3)
    assert set(np.unique(fm.codes3(p3, K, N)).tolist()) == set(range(8))
