"""CPU oracle for decode attention over a symbolic KV length -- TEST
INFRASTRUCTURE ONLY (rules of ``oracle/__init__.py``: only tests, smoke() and
bench.py's CPU legs may use it; it shares no code with the product package).

SURVEY §8(f) F4 / PAPER P:102 ("the KV-cache context length" is a dynamic
dimension), P:641 (single-batch decode of Llama-2): one new query token per
sequence attends over that sequence's cached keys and values.  Written out
plainly in float64 (DESIGN.md §3 reading 21):

  q        fp16 [batch][Hq][D]
  k, v     fp16 [batch][Hkv][L_max][D]   (cache; positions >= len[b] unused)
  len      int  [batch]                   (the symbolic KV length of each sequence)
  group    h -> kv head h // (Hq / Hkv)   (grouped-query attention; Hq = Hkv is MHA)
  s_j      = (q[b,h] . k[b,g,j]) / sqrt(D)              j < len[b]
  p_j      = exp(s_j - max_j s) / sum_j exp(s_j - max_j s)
  out[b,h] = sum_j p_j v[b,g,j]                          (0 when len[b] == 0)

and the KV append of the new token's key and value at position pos[b].
"""
from __future__ import annotations

import numpy as np


def _f(bits):
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


def attention_decode(q_bits, k_bits, v_bits, lens, n_kv_heads: int) -> np.ndarray:
    """float64 out [batch][Hq][D]."""
    q = _f(q_bits)
    k = _f(k_bits)
    v = _f(v_bits)
    batch, hq, d = q.shape
    group = hq // n_kv_heads
    out = np.zeros((batch, hq, d))
    for b in range(batch):
        L = int(lens[b])
        if L == 0:
            continue
        for h in range(hq):
            g = h // group
            s = k[b, g, :L, :] @ q[b, h, :] / np.sqrt(d)
            p = np.exp(s - s.max())
            p /= p.sum()
            out[b, h, :] = p @ v[b, g, :L, :]
    return out


def kv_append(k_cache_bits, v_cache_bits, k_new_bits, v_new_bits, pos):
    """Copies of the caches with [b, :, pos[b], :] = the new key / value."""
    kc = np.array(k_cache_bits, dtype=np.uint16, copy=True)
    vc = np.array(v_cache_bits, dtype=np.uint16, copy=True)
    for b in range(kc.shape[0]):
        kc[b, :, int(pos[b]), :] = k_new_bits[b]
        vc[b, :, int(pos[b]), :] = v_new_bits[b]
    return kc, vc
