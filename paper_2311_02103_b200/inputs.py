"""Seeded synthetic inputs -- the ONE module both the oracle tests and the
CUDA path's tests/bench draw from.

It holds none of the method's arithmetic (no dequantization, no matmul): it
only draws random numbers and encodes them in the q4f16 storage format
(readings 1-4: unsigned 4-bit codes, implicit zero point 7,
one fp16 scale per 32 consecutive k, eight codes per little-endian uint32,
``packed_w uint32[N][K/8]``, ``scales fp16[N][K/32]``, ``x fp16[n][K]``).

Recipes:
  realistic  W_true ~ N(0, 0.02^2), quantised per 32-group with
             s = fp16(max|w|/7), q = clamp(rne(w/s) + 7, 0, 14), q = 7 if s == 0
             (test-data quantiser, not on the hot path); x ~ N(0,1) -> fp16.
  stress     codes uniform on 0..15 (incl. 15), scales uniform in
             [2^-10, 2^-6] -> fp16; x ~ U(-1, 1) -> fp16.
RNG: numpy PCG64.  Weight seed = 1000*config + matrix index; x seed = 7 + n.
fp16 values are returned as uint16 bit patterns (numpy float16 .view).
"""
from __future__ import annotations

import numpy as np

GROUP = 32          # codes per scale (reading 2)
CODES_PER_WORD = 8  # reading 3


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """codes uint8 [N][K] (values 0..15) -> uint32 [N][K/8]; element k sits at
    bits 4*(k mod 8) of word k/8 (low nibble first)."""
    codes = np.asarray(codes, dtype=np.uint32)
    N, K = codes.shape
    assert K % CODES_PER_WORD == 0
    c = codes.reshape(N, K // CODES_PER_WORD, CODES_PER_WORD)
    words = np.zeros((N, K // CODES_PER_WORD), dtype=np.uint32)
    for t in range(CODES_PER_WORD):
        words |= c[:, :, t] << np.uint32(4 * t)
    return words


def f16_bits(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float16).view(np.uint16)


def realistic_weights(seed: int, K: int, N: int, std: float = 0.02,
                      chunk_rows: int = 2048):
    """(packed_w uint32[N][K/8], scales uint16[N][K/32]) from quantised
    N(0, std^2) weights.  Generated in row chunks to bound host memory."""
    assert K % GROUP == 0
    g = rng(seed)
    packed = np.empty((N, K // CODES_PER_WORD), dtype=np.uint32)
    scales = np.empty((N, K // GROUP), dtype=np.uint16)
    for r0 in range(0, N, chunk_rows):
        r1 = min(N, r0 + chunk_rows)
        w = g.standard_normal((r1 - r0, K), dtype=np.float32) * np.float32(std)
        wg = w.reshape(r1 - r0, K // GROUP, GROUP)
        s16 = (np.abs(wg).max(axis=2) / np.float32(7.0)).astype(np.float16)
        s32 = s16.astype(np.float32)
        safe = np.where(s32 == 0, np.float32(1.0), s32)
        q = np.rint(wg / safe[:, :, None]) + np.float32(7.0)
        q = np.clip(q, 0, 14)
        q = np.where((s32 == 0)[:, :, None], np.float32(7.0), q)
        packed[r0:r1] = pack_codes(q.reshape(r1 - r0, K).astype(np.uint8))
        scales[r0:r1] = s16.view(np.uint16)
    return packed, scales


def stress_weights(seed: int, K: int, N: int):
    """Uniform random codes 0..15 and scales uniform in [2^-10, 2^-6]."""
    assert K % GROUP == 0
    g = rng(seed)
    packed = g.integers(0, 2**32, size=(N, K // CODES_PER_WORD), dtype=np.uint64)
    packed = packed.astype(np.uint32)
    s = g.uniform(2.0**-10, 2.0**-6, size=(N, K // GROUP))
    return packed, f16_bits(s)


def activations(seed: int, n: int, K: int, dist: str = "normal") -> np.ndarray:
    """x as fp16 bits [n][K]."""
    g = rng(seed)
    if dist == "normal":
        x = g.standard_normal((n, K), dtype=np.float32)
    elif dist == "uniform":
        x = g.uniform(-1.0, 1.0, size=(n, K)).astype(np.float32)
    else:
        raise ValueError(dist)
    return f16_bits(x)


def weights(kind: str, seed: int, K: int, N: int):
    if kind == "realistic":
        return realistic_weights(seed, K, N)
    if kind == "stress":
        return stress_weights(seed, K, N)
    raise ValueError(kind)


# Llama-2 linear-layer shapes (K = in_features, N = out_features) per layer,
# SURVEY §8(d) configs c2/c4/c5.  Name -> list of (name, K, N, count/layer).
LLAMA_SETS = {
    "llama2-7b": dict(layers=32, mats=[("q", 4096, 4096), ("k", 4096, 4096),
                                        ("v", 4096, 4096), ("o", 4096, 4096),
                                        ("gate", 4096, 11008), ("up", 4096, 11008),
                                        ("down", 11008, 4096)],
                      lm_head=(4096, 32000)),
    "llama2-13b": dict(layers=40, mats=[("q", 5120, 5120), ("k", 5120, 5120),
                                         ("v", 5120, 5120), ("o", 5120, 5120),
                                         ("gate", 5120, 13824), ("up", 5120, 13824),
                                         ("down", 13824, 5120)],
                       lm_head=(5120, 32000)),
    "llama2-70b": dict(layers=80, mats=[("q", 8192, 8192), ("k", 8192, 1024),
                                         ("v", 8192, 1024), ("o", 8192, 8192),
                                         ("gate", 8192, 28672), ("up", 8192, 28672),
                                         ("down", 28672, 8192)],
                       lm_head=(8192, 32000)),
}


def q4_bytes(K: int, N: int) -> int:
    """Stored bytes of one q4f16 weight: K*N/2 codes + K*N/32*2 scales."""
    return K * N // 2 + (K // GROUP) * N * 2
