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
