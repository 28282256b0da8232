"""Pins of oracle/attention.py (decode attention over a symbolic KV length,
SURVEY §8(f) F4; reading 21) against closed forms and a
pure-Python brute force."""
import math

import numpy as np

from oracle import attention as oa


def f16(a):
    return np.asarray(a, dtype=np.float16).view(np.uint16)


def test_single_key_returns_its_value():
    rng = np.random.default_rng(0)
    q = f16(rng.standard_normal((1, 2, 128)))
    k = f16(rng.standard_normal((1, 2, 8, 128)))
    v = f16(rng.standard_normal((1, 2, 8, 128)))
    out = oa.attention_decode(q, k, v, [1], n_kv_heads=2)
    assert np.array_equal(out[0], v[0, :, 0, :].view(np.float16).astype(np.float64))


def test_zero_query_averages_values_and_empty_is_zero():
    rng = np.random.default_rng(1)
    q = f16(np.zeros((2, 4, 128)))
    k = f16(rng.standard_normal((2, 1, 16, 128)))
    v = f16(rng.standard_normal((2, 1, 16, 128)))
    out = oa.attention_decode(q, k, v, [5, 0], n_kv_heads=1)
    want = v[0, 0, :5, :].view(np.float16).astype(np.float64).mean(axis=0)
    for h in range(4):
        assert np.allclose(out[0, h], want, rtol=0, atol=1e-15)
    assert np.all(out[1] == 0)


def test_gqa_group_mapping():
    # kv head g holds values == g everywhere: query head h must read kv head h // (Hq/Hkv)
    hq, hkv, L = 8, 2, 4
    q = f16(np.random.default_rng(2).standard_normal((1, hq, 128)))
    k = f16(np.random.default_rng(3).standard_normal((1, hkv, L, 128)))
    v = f16(np.broadcast_to(np.arange(hkv, dtype=np.float64)[None, :, None, None], (1, hkv, L, 128)))
    out = oa.attention_decode(q, k, v, [L], n_kv_heads=hkv)
    for h in range(hq):
        assert np.allclose(out[0, h], h // (hq // hkv), rtol=0, atol=1e-12)


def test_brute_force_python():
    rng = np.random.default_rng(4)
    hq, hkv, L, d = 4, 2, 7, 128
    q = f16(rng.standard_normal((1, hq, d)))
    k = f16(rng.standard_normal((1, hkv, 9, d)))
    v = f16(rng.standard_normal((1, hkv, 9, d)))
    out = oa.attention_decode(q, k, v, [L], n_kv_heads=hkv)
    qf, kf, vf = (a.view(np.float16).astype(float) for a in (q, k, v))
    for h in range(hq):
        g = h // 2
        s = [sum(qf[0, h, i] * kf[0, g, j, i] for i in range(d)) / math.sqrt(d) for j in range(L)]
        m = max(s)
        e = [math.exp(x - m) for x in s]
        tot = sum(e)
        for i in range(0, d, 17):
            want = sum(e[j] / tot * vf[0, g, j, i] for j in range(L))
            assert abs(out[0, h, i] - want) <= 1e-12 * max(1.0, abs(want))


def test_kv_append():
    kc = np.zeros((2, 3, 5, 128), dtype=np.uint16)
    vc = np.ones((2, 3, 5, 128), dtype=np.uint16)
    kn = np.full((2, 3, 128), 7, dtype=np.uint16)
    vn = np.full((2, 3, 128), 9, dtype=np.uint16)
    k2, v2 = oa.kv_append(kc, vc, kn, vn, [4, 0])
    assert np.all(k2[0, :, 4] == 7) and np.all(k2[1, :, 0] == 7)
    assert np.all(v2[0, :, 4] == 9) and np.all(v2[1, :, 0] == 9)
    assert np.all(k2[0, :, :4] == 0) and np.all(v2[1, :, 1:] == 1)
