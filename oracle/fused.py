"""CPU oracle for the fused neighbours of the q4 matmul -- TEST INFRASTRUCTURE ONLY.

Same rules as the rest of ``oracle/`` (see ``oracle/__init__.py``): only
tests, ``__graft_entry__.smoke()`` and bench.py's CPU legs may use it; it
shares no code with the product package.

Fusion preserves the semantics of the unfused program (FuseOps /
FuseTensorIR merge the element-wise producers and consumers of a matmul into
one tensor program).  The unfused Llama decoder block passes fp16 tensors
between kernels, so each operator here is that kernel written out plainly in
numpy, fp16 at every tensor boundary, float64 inside where the unfused kernel
would compute in float32 (DESIGN.md §3 readings 16-18):

  rmsnorm_x(x, gamma, eps)
      r_t     = 1 / sqrt(mean_k x[t,k]^2 + eps)                    (float64)
      h       = fp16_RNE(x * r_t)                                   (the cast back to fp16)
      xn      = fp16_RNE(h * gamma)                                 (fp16 x fp16 product, one rounding)
  silu_mul(r, pairs)    r: the matmul's float64 sums over interleaved rows
      g, u    = fp16_RNE(r[:, 0::2]), fp16_RNE(r[:, 1::2])          (matmul output is fp16)
      y_ref   = silu(g) * u,  silu(g) = g / (1 + exp(-g))           (float64, compared with tolerance)
  residual(v, res)      v: fp16 output so far (bits) or its float64 reference
      y_ref   = v + res                                             (float64)

The matmul itself is ``oracle.matmul_f64`` (plain C, fp64).
"""
from __future__ import annotations

import numpy as np


def _f16(bits: np.ndarray) -> np.ndarray:
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float64)


def _bits(v: np.ndarray) -> np.ndarray:
    return np.asarray(v, dtype=np.float64).astype(np.float16).view(np.uint16)


def rmsnorm_x(x_bits: np.ndarray, gamma_bits: np.ndarray, eps: float) -> np.ndarray:
    """Llama RMSNorm of fp16 rows x [n, K] with fp16 gamma [K] -> fp16 bits [n, K]."""
    x = _f16(x_bits)
    g = _f16(gamma_bits)
    ms = np.mean(x * x, axis=1, keepdims=True)
    r = 1.0 / np.sqrt(ms + float(eps))
    h = (x * r).astype(np.float16).astype(np.float64)      # one RNE rounding of x * r_t
    return _bits(h * g)                                      # exact product, one RNE rounding


def silu(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    with np.errstate(over="ignore"):
        return v / (1.0 + np.exp(-v))


def silu_mul(r: np.ndarray) -> np.ndarray:
    """r: float64 matmul sums [n, N] over interleaved (gate, up) rows -> float64 y_ref [n, N/2]."""
    r = np.asarray(r, dtype=np.float64)
    g = r[:, 0::2].astype(np.float16).astype(np.float64)
    u = r[:, 1::2].astype(np.float16).astype(np.float64)
    return silu(g) * u


def residual(v: np.ndarray, res_bits: np.ndarray, v_is_bits: bool = False) -> np.ndarray:
    """y_ref = v + residual (float64); v is fp16-rounded first (the unfused
    matmul / SiLU-mul output is an fp16 tensor)."""
    vv = _f16(v) if v_is_bits else np.asarray(v, dtype=np.float64).astype(np.float16).astype(np.float64)
    return vv + _f16(res_bits)


def interleave_rows(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Rows of a and b alternated: out[2j] = a[j], out[2j+1] = b[j] (the
    gate/up pairing of RELAX_OP_SILU_MUL)."""
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    out = np.empty((2 * a.shape[0],) + a.shape[1:], dtype=a.dtype)
    out[0::2] = a
    out[1::2] = b
    return out
