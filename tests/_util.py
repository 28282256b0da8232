"""Shared test helpers: device transfer and the north-star tolerance check.

Tolerance (BASELINE.json north_star; definitions DESIGN.md §3 reading 10):
  rel_F   = ||y - r||_F / ||r||_F                      <= 2e-3
  max_rel = max_ij |y - r| / max(|r_ij|, rms(r_i,:))   <= 1e-2
where r is the oracle's fp64 sum over the fp16-rounded weights.  If r is
identically zero, y must be exactly (signed) zero.
"""
import numpy as np

REL_F = 2e-3
MAX_REL = 1e-2


def dev_weights(packed, scales):
    import torch
    pw = torch.from_numpy(np.ascontiguousarray(packed).view(np.int32)).cuda()
    sc = torch.from_numpy(np.ascontiguousarray(scales).view(np.float16)).cuda()
    return pw, sc


def dev_x(x_bits):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x_bits).view(np.float16)).cuda()


def host_bits(t):
    return t.detach().cpu().contiguous().view(__import__("torch").int16).numpy().view(np.uint16)


def tol_stats(y_bits, r):
    return tol_stats_f(np.asarray(y_bits, dtype=np.uint16).view(np.float16).astype(np.float64), r)


def tol_stats_f(y, r):
    y = np.asarray(y, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    diff = y - r
    nr = np.linalg.norm(r)
    rel_f = np.linalg.norm(diff) / nr if nr > 0 else float(np.linalg.norm(diff))
    rms = np.sqrt(np.mean(r * r, axis=1, keepdims=True))
    denom = np.maximum(np.abs(r), rms)
    with np.errstate(invalid="ignore", divide="ignore"):
        rel = np.where(denom > 0, np.abs(diff) / denom, np.abs(diff))
    return {"rel_f": float(rel_f), "max_rel": float(np.max(rel)) if rel.size else 0.0,
            "finite": bool(np.all(np.isfinite(y)))}


def assert_within_tol(y_bits, r, what=""):
    st = tol_stats(y_bits, r)
    assert st["finite"], f"{what}: non-finite output"
    if np.all(np.asarray(r) == 0):
        y = np.asarray(y_bits, dtype=np.uint16)
        assert np.all((y & 0x7FFF) == 0), f"{what}: r == 0 but y != 0"
        return st
    assert st["rel_f"] <= REL_F, f"{what}: rel_F {st['rel_f']:.3e} > {REL_F}"
    assert st["max_rel"] <= MAX_REL, f"{what}: max_rel {st['max_rel']:.3e} > {MAX_REL}"
    return st


def assert_within_tol_f(y, r, what=""):
    """assert_within_tol for outputs already decoded to float64 (y != 0 where r == 0 fails)."""
    st = tol_stats_f(y, r)
    assert st["finite"], f"{what}: non-finite output"
    if np.all(np.asarray(r) == 0):
        assert np.all(np.asarray(y) == 0), f"{what}: r == 0 but y != 0"
        return st
    assert st["rel_f"] <= REL_F, f"{what}: rel_F {st['rel_f']:.3e} > {REL_F}"
    assert st["max_rel"] <= MAX_REL, f"{what}: max_rel {st['max_rel']:.3e} > {MAX_REL}"
    return st
