"""CPU oracle for the q4 storage-format variants -- TEST INFRASTRUCTURE ONLY.

Same rules as the rest of ``oracle/`` (see ``oracle/__init__.py``): only tests,
``__graft_entry__.smoke()`` and bench.py's CPU legs may use it; it shares no
code with the product package.

SURVEY §8(f) F3 / PAPER P:442-443 ("lift out quantization and layout
transforms in tensor programs to enable pre-computation"): a checkpoint may
store its int4 weights in another layout or with another group size; the
product converts it ONCE (relax_q4_repack) into the kernel-native format
(DESIGN.md §3 readings 1-4 and 19-20).  Each source format is defined here by
its dequantized weight, written out plainly:

  layout "nk" (native):  packed[j][k/8] holds code q(k, j) at bits 4*(k mod 8);
                          scales[j][k/G]
  layout "kn":            packed[k/8][j] holds code q(k, j) at bits 4*(k mod 8)
                          (the per-column packing along K of GPTQ-style
                          checkpoints); scales[k/G][j]
  W(k, j) = fp16_RNE((q(k, j) - 7) * s(k/G, j)),  G in {32, 64, 128}

and the native format is G = 32, layout "nk".  3-bit weights (the
iPhone runs Llama-2-7B "in 3-bit"; reading 20):

  layout "nk3":           packed[j][3 g .. 3 g + 2] holds the 32 codes of
                          group g of column j, code i at bits 3 i .. 3 i + 2
                          of the 96-bit little-endian word triple (codes 10
                          and 21 straddle the word boundaries); scales[j][k/G]
  W(k, j) = fp16_RNE((q3(k, j) - 3) * s(k/G, j)),  q3 in [0, 7]

whose native form is q4 = q3 + 4 (so q4 - 7 == q3 - 3: the same W).  ``to_native`` is the plain
definition of the conversion: the codes are moved, not changed, and each
32-code group takes the scale of the G-group that contains it, so the
converted weight dequantizes to the same W bit for bit.
"""
from __future__ import annotations

import numpy as np

LAYOUTS = ("nk", "kn")          # 4-bit layouts; "nk3" is the 3-bit one
GROUPS = (32, 64, 128)


def codes(packed: np.ndarray, K: int, N: int, layout: str) -> np.ndarray:
    """q(k, j) as uint8 [N][K] (column j of W is row j)."""
    p = np.asarray(packed, dtype=np.uint32)
    q = np.empty((N, K), dtype=np.uint8)
    for k in range(K):
        word = p[:, k // 8] if layout == "nk" else p[k // 8, :]
        q[:, k] = (word >> np.uint32(4 * (k % 8))) & np.uint32(0xF)
    return q


def codes3(packed: np.ndarray, K: int, N: int) -> np.ndarray:
    """q3(k, j) as uint8 [N][K] from the "nk3" words [N][3 K/32]."""
    p = np.asarray(packed, dtype=np.uint64)
    q = np.empty((N, K), dtype=np.uint8)
    for g in range(K // 32):
        for i in range(32):
            bit = 3 * i                                   # within the group's 96 bits
            w, off = 3 * g + bit // 32, bit % 32
            v = p[:, w] >> np.uint64(off)
            if off > 29:                                  # the code continues in the next word
                v = v | (p[:, w + 1] << np.uint64(32 - off))
            q[:, 32 * g + i] = (v & np.uint64(7)).astype(np.uint8)
    return q


def dequant3(packed, scales, K: int, N: int, group: int) -> np.ndarray:
    """W as fp16 bits [N][K] of an "nk3" weight: fp16_RNE((q3 - 3) * s)."""
    q = codes3(packed, K, N).astype(np.float32) - np.float32(3.0)
    s = scale_of(scales, K, N, "nk", group).view(np.float16).astype(np.float32)
    return (q * s).astype(np.float16).view(np.uint16)


def pack4(q: np.ndarray) -> np.ndarray:
    """Native words [N][K/8] of 4-bit codes q [N][K]: code k at bits 4 (k mod 8)."""
    N, K = q.shape
    out = np.zeros((N, K // 8), dtype=np.uint32)
    for k in range(K):
        out[:, k // 8] |= q[:, k].astype(np.uint32) << np.uint32(4 * (k % 8))
    return out


def scale_of(scales: np.ndarray, K: int, N: int, layout: str, group: int) -> np.ndarray:
    """s(k/G, j) as fp16 bits [N][K] (one entry per weight)."""
    s = np.asarray(scales, dtype=np.uint16)
    per_group = s if layout == "nk" else s.T                   # [N][K/G]
    return np.repeat(per_group, group, axis=1)[:, :K]


def dequant(packed, scales, K: int, N: int, layout: str, group: int) -> np.ndarray:
    """W as fp16 bits [N][K]: one RNE rounding of the exact product (q - 7) * s
    (exact in float32: <= 4 + 11 significant bits)."""
    q = codes(packed, K, N, layout).astype(np.float32) - np.float32(7.0)
    s = scale_of(scales, K, N, layout, group).view(np.float16).astype(np.float32)
    return (q * s).astype(np.float16).view(np.uint16)


def to_native(packed, scales, K: int, N: int, layout: str, group: int):
    """The native (layout "nk", G = 32) packed codes and scales holding the same W."""
    p = np.asarray(packed, dtype=np.uint32)
    s = np.asarray(scales, dtype=np.uint16)
    if layout == "nk3":
        pk = pack4(codes3(p, K, N) + np.uint8(4))               # q4 = q3 + 4
        return np.ascontiguousarray(pk), np.ascontiguousarray(np.repeat(s, group // 32, axis=1))
    pk = p if layout == "nk" else p.T                           # same words, transposed
    sg = s if layout == "nk" else s.T                           # [N][K/G]
    sc = np.repeat(sg, group // 32, axis=1)                     # [N][K/32]
    return np.ascontiguousarray(pk), np.ascontiguousarray(sc)
