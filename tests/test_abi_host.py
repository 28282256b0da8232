"""Host-side tests of the C-ABI (no GPU needed): the library loads, exports
every symbol include/relax_q4.h declares, validates arguments before any CUDA
call ("never a wrong answer"), and its upper-bound workspace plan
is sound."""
import ctypes
import os
import random
import re

import pytest

from paper_2311_02103_b200 import build, ops

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return ops.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "relax_q4.h")).read()
    return sorted(set(re.findall(r"RELAX_API\s+[\w\s\*]+?\b(relax_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) == 10
    assert sorted(ops.EXPORTS) == syms
    for s in syms:
        assert hasattr(L, s), s
    assert ops.version().startswith("relax_q4")


def test_status_strings(L):
    for code, name in ops.STATUS.items():
        assert L.relax_status_str(code).decode().startswith(name)
    assert L.relax_status_str(99).decode() == "RELAX_ERR_UNKNOWN"


A = 0x10000          # fake, 16-byte aligned, never dereferenced: validation
MB = 1 << 20         # precedes every CUDA call


def call(L, x=A, n=1, K=256, N=256, w=A + 8 * MB, s=A + 16 * MB, y=A + 24 * MB, ws=0, wsb=0):
    return L.relax_q4_matmul_ws(x, n, K, N, w, s, y, ws, wsb, None)


def test_validation_codes(L):
    assert call(L, n=-1) == 1
    assert call(L, K=0) == 1
    assert call(L, N=0) == 1
    assert call(L, x=0) == 1
    assert call(L, y=0) == 1
    assert call(L, w=0) == 1
    assert call(L, ws=0, wsb=64) == 1
    assert call(L, K=100) == 2                       # K % 32 != 0
    assert call(L, n=0, x=0, y=0) == 0               # n == 0: no-op
    assert call(L, x=A + 2) == 3                     # misaligned
    assert call(L, y=A + 8 * MB + 8) == 3
    assert call(L, y=A + 8 * MB) == 4                # y overlaps packed_w
    assert call(L, y=A + 100) in (3, 4)
    assert call(L, y=A + 112) == 4                   # y overlaps x (aligned)
    assert call(L, ws=A + 24 * MB, wsb=1024) == 4    # workspace overlaps y
    # valid arguments reach the device check: there is no GPU here
    assert call(L) == 6
    assert L.relax_q4_matmul(A, 4, 256, 256, A + 8 * MB, A + 16 * MB, A + 24 * MB, None) == 6
    assert L.relax_q4_dequant(A, A + MB, 256, 256, A + 8 * MB, None) == 6
    assert L.relax_q4_dequant(A, A + MB, 256, 256, A, None) == 4
    assert L.relax_q4_dequant(A, A + MB, 250, 256, A + 8 * MB, None) == 2
    assert L.relax_q4_dequant(A, A + MB, 256, 0, 0, None) == 0


def test_workspace_too_small_is_reported(L):
    # a forced split-K through the workspace (RELAX_FLAG_SPLIT_WORKSPACE) needs
    # split * n * N * 4 B + tickets: a 16-byte workspace is too small
    assert L.relax_q4_matmul_ex(A, 16, 8192, 1024, A + 8 * MB, A + 16 * MB, A + 64 * MB,
                                A + 128 * MB, 16, 2, 8, 16, 2, None) == 5
    # the automatic schedule splits K inside a thread-block cluster (DSMEM
    # reduction): no workspace at all, so a workspace-free call proceeds
    sched = ops.query_schedule(16, 8192, 1024)
    assert sched["variant"] == "tc" and sched["split_k"] > 1 and sched["ws_bytes"] == 0
    assert call(L, n=16, K=8192, N=1024, y=A + 64 * MB) == 6
    assert ops.query_schedule(16, 4096, 4096)["ws_bytes"] == 0
    # forced TC on a K that is not a multiple of 256
    assert L.relax_q4_matmul_ex(A, 16, 4128, 256, A + 8 * MB, A + 16 * MB, A + 64 * MB, 0, 0,
                                2, 0, 0, 0, None) == 2


def test_plan_invalid(L):
    out = ctypes.c_size_t()
    assert L.relax_plan_workspace(-1, 256, 256, ctypes.byref(out)) == 1
    assert L.relax_plan_workspace(8, 0, 256, ctypes.byref(out)) == 1
    assert L.relax_plan_workspace(8, 256, 256, None) == 1
    assert L.relax_plan_workspace(8, 100, 256, ctypes.byref(out)) == 2


SHAPES = [(256, 256), (4096, 4096), (4096, 11008), (11008, 4096), (4096, 32000),
          (5120, 13824), (8192, 1024), (28672, 8192), (8192, 28672), (1024, 128), (96, 64)]


@pytest.mark.parametrize("K,N", SHAPES)
def test_plan_soundness_random_bindings(K, N):
    """S:467 plan soundness: every n <= n_max needs <= plan(n_max) bytes."""
    rng = random.Random(K * 31 + N)
    for n_max in (1, 16, 100, 4096):
        bound = ops.plan_workspace(n_max, K, N)
        for _ in range(250):
            n = rng.randint(1, n_max)
            assert ops.query_schedule(n, K, N)["ws_bytes"] <= bound


@pytest.mark.parametrize("K,N", SHAPES[:6])
def test_plan_monotone_in_n_max(K, N):
    prev = 0
    for n_max in (0, 1, 2, 8, 16, 17, 64, 100, 256, 1000, 4096, 100000):
        b = ops.plan_workspace(n_max, K, N)
        assert b >= prev
        prev = b


def test_plan_is_exact_max():
    K, N, n_max = 4096, 4096, 300
    m = max(ops.query_schedule(n, K, N)["ws_bytes"] for n in range(1, n_max + 1))
    assert ops.plan_workspace(n_max, K, N) == m


def test_dispatch_shape_specialisation():
    """n decides the variant: GEMV at decode, tensor cores for
    prefill; K % 256 != 0 keeps GEMV at any n."""
    assert ops.query_schedule(1, 4096, 4096)["variant"] == "gemv"
    assert ops.query_schedule(2, 4096, 4096)["variant"] == "gemv"
    assert ops.query_schedule(3, 4096, 4096)["variant"] == "tc"
    s = ops.query_schedule(4096, 4096, 4096)
    assert s["variant"] == "tc" and s["tile"] in (128, 256) and s["split_k"] == 1
    assert ops.query_schedule(512, 4128, 4096)["variant"] == "gemv"
    for n in (17, 100, 1000):
        s = ops.query_schedule(n, 4096, 11008)
        assert s["variant"] == "tc" and s["tile"] >= min(n, 16)


# ------------------------------------------------------------- fused neighbours
def fcall(L, ops_=0, eps=1e-5, gamma=A + 32 * MB, res=0, x=A, n=1, K=256, N=256, w=A + 8 * MB,
          s=A + 16 * MB, y=A + 24 * MB, ws=0, wsb=0):
    fz = ops.Fusion(ops_, eps, gamma or None, res or None)
    return L.relax_q4_matmul_fused(x, n, K, N, w, s, y, ctypes.byref(fz), ws, wsb, None)


def test_fused_validation_codes(L):
    R, S, Q = ops.OP_RMSNORM_X, ops.OP_SILU_MUL, ops.OP_RESIDUAL
    assert fcall(L, ops_=8) == 1                                  # unknown op bit
    assert fcall(L, ops_=R, K=96) == 2                            # fused ops need K % 256 == 0
    assert fcall(L, ops_=S, N=255) == 2                           # SiLU-mul pairs need N even
    assert fcall(L, ops_=R, gamma=0) == 1                         # RMSNorm without gamma
    assert fcall(L, ops_=R, eps=-1.0) == 1
    assert fcall(L, ops_=R, eps=float("nan")) == 1
    assert fcall(L, ops_=Q, res=0) == 1                           # residual without pointer
    assert fcall(L, ops_=R, gamma=A + 32 * MB + 8) == 3           # misaligned gamma
    assert fcall(L, ops_=Q, res=A + 24 * MB + 16) == 4            # residual partially overlapping y
    assert fcall(L, ops_=R, gamma=A + 24 * MB) == 4               # y overlapping gamma
    assert fcall(L, ops_=Q, res=A + 24 * MB) == 6                 # in-place residual (res == y) is legal
    assert fcall(L, ops_=R | S | Q, res=A + 40 * MB) == 6         # valid: reaches the device check
    assert fcall(L, ops_=R, n=64) == 5                            # TC path normalises into the workspace
    assert fcall(L, ops_=R, n=0, x=0, y=0) == 0                   # n == 0: no-op
    assert fcall(L, ops_=0, K=100) == 2                           # ops == 0: plain matmul validation


def test_fused_workspace_plan(L):
    R = ops.OP_RMSNORM_X
    assert ops.plan_workspace_fused(2, 4096, 4096, R) == 0        # decode GEMV normalises in registers
    assert ops.plan_workspace_fused(64, 4096, 4096, 0) == ops.plan_workspace(64, 4096, 4096)
    assert ops.plan_workspace_fused(64, 4096, 4096, R) >= 64 * 4096 * 2
    assert ops.plan_workspace_fused(100000, 4096, 4096, R) >= 100000 * 4096 * 2
    with pytest.raises(ops.RelaxError):
        ops.plan_workspace_fused(4, 4096, 4095 * 2 + 1, ops.OP_SILU_MUL)
    # plan soundness: every n <= n_max fits
    for n_max in (1, 3, 17, 300):
        nb = ops.plan_workspace_fused(n_max, 4096, 11008, R)
        for n in range(1, n_max + 1, max(1, n_max // 7)):
            assert fcall(L, ops_=R, n=n, K=4096, N=11008, w=A + 64 * MB, s=A + 128 * MB, y=A + 256 * MB,
                         gamma=A + 512 * MB, ws=A + 1024 * MB, wsb=nb) == 6


@pytest.mark.parametrize("n", [3, 8, 16, 32, 64, 128, 512])
@pytest.mark.parametrize("K,N", [(4096, 4096), (4096, 11008), (11008, 4096), (4096, 12288), (4096, 22016),
                                 (8192, 1024), (8192, 28672)])
def test_split_clusters_fit_one_wave(n, K, N):
    """Automatic split-K never asks for more clusters than one wave holds on a
    B200 (profiles/tc_waves_r01.txt): 4096 x 12288 at n = 8 takes
    s = 2, not the 3 that two CTAs per SM alone would suggest."""
    cap2 = {1: 296, 2: 148, 3: 93, 4: 71, 5: 56, 6: 45, 7: 37, 8: 33}
    cap1 = {1: 148, 2: 74, 3: 45, 4: 33, 5: 26, 6: 22, 7: 15, 8: 15}
    s = ops.query_schedule(n, K, N)
    if s["variant"] != "tc" or s["split_k"] == 1:
        return
    tiles = -(-N // 128) * -(-n // s["tile"])
    cap = (cap2 if s["tile"] <= 64 else cap1)[s["split_k"]]
    assert tiles <= cap, (s, tiles, cap)
    if (n, K, N) == (8, 4096, 12288):
        assert s["split_k"] == 2
