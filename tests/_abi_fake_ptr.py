"""Fake-pointer validation of the C-ABI, run by tests/test_abi_host.py in a
subprocess with CUDA_VISIBLE_DEVICES="" (so valid arguments stop at the device
check, RELAX_ERR_DEVICE = 6, and nothing is launched on the fake addresses).

Validation is O(1) and precedes every CUDA call (include/relax_q4.h; SPEC
S:629 "never a wrong answer"): null pointers / bad sizes -> 1, K % 32 -> 2,
misalignment -> 3, aliasing -> 4, short workspace -> 5."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_02103_b200 import ops  # noqa: E402

A = 0x10000          # fake, 16-byte aligned, never dereferenced
MB = 1 << 20


def call(L, x=A, n=1, K=256, N=256, w=A + 8 * MB, s=A + 16 * MB, y=A + 24 * MB, ws=0, wsb=0):
    return L.relax_q4_matmul_ws(x, n, K, N, w, s, y, ws, wsb, None)


def validation_codes(L):
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
    # valid arguments reach the device check: no device is visible here
    assert call(L) == 6
    assert L.relax_q4_matmul(A, 4, 256, 256, A + 8 * MB, A + 16 * MB, A + 24 * MB, None) == 6
    assert L.relax_q4_dequant(A, A + MB, 256, 256, A + 8 * MB, None) == 6
    assert L.relax_q4_dequant(A, A + MB, 256, 256, A, None) == 4
    assert L.relax_q4_dequant(A, A + MB, 250, 256, A + 8 * MB, None) == 2
    assert L.relax_q4_dequant(A, A + MB, 256, 0, 0, None) == 0
    # very wide outputs plan a schedule that fits and reach the device check
    assert L.relax_q4_matmul(A, 1, 16384, 128256, A + 8 * MB, A + 2048 * MB, A + 4096 * MB, None) == 6


def workspace_too_small(L):
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


def plan_invalid(L):
    out = ctypes.c_size_t()
    assert L.relax_plan_workspace(-1, 256, 256, ctypes.byref(out)) == 1
    assert L.relax_plan_workspace(8, 0, 256, ctypes.byref(out)) == 1
    assert L.relax_plan_workspace(8, 256, 256, None) == 1
    assert L.relax_plan_workspace(8, 100, 256, ctypes.byref(out)) == 2


def fcall(L, ops_=0, eps=1e-5, gamma=A + 32 * MB, res=0, x=A, n=1, K=256, N=256, w=A + 8 * MB,
          s=A + 16 * MB, y=A + 24 * MB, ws=0, wsb=0):
    fz = ops.Fusion(ops_, eps, gamma or None, res or None)
    return L.relax_q4_matmul_fused(x, n, K, N, w, s, y, ctypes.byref(fz), ws, wsb, None)


def fused_validation_codes(L):
    R, S, Q = ops.OP_RMSNORM_X, ops.OP_SILU_MUL, ops.OP_RESIDUAL
    assert fcall(L, ops_=16) == 1                                 # unknown op bit
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
    # a SiLU-mul decode call on a row pair layout too wide for the streamed
    # kernel takes the tensor path (needs no workspace without RMSNorm)
    assert fcall(L, ops_=S, n=1, K=16384, N=2 * 128256, w=A + 64 * MB, s=A + 4096 * MB, y=A + 8192 * MB) == 6


def kv_append_validation(L):
    """RELAX_OP_KV_APPEND (the KV append fused into the q/k/v epilogue)."""
    KV = ops.OP_KV_APPEND
    C = A + 512 * MB

    def kcall(n=1, K=256, N=1024, kc=C, vc=C + 64 * MB, pos=C + 128 * MB, lmax=64, heads=2, row0=256, o=0):
        fz = ops.Fusion(KV | o, 1e-5, (A + 32 * MB) if o & ops.OP_RMSNORM_X else None, None)
        fz.k_cache, fz.v_cache, fz.kv_pos = kc, vc, pos
        fz.kv_len_max, fz.kv_heads, fz.kv_row0 = lmax, heads, row0
        return L.relax_q4_matmul_fused(A, n, K, N, A + 8 * MB, A + 16 * MB, A + 24 * MB, ctypes.byref(fz), 0, 0,
                                       None)
    assert kcall() == 6                                           # valid: device check
    assert kcall(o=ops.OP_RMSNORM_X) == 6
    assert kcall(kc=0) == 1 and kcall(pos=0) == 1 and kcall(heads=0) == 1 and kcall(lmax=0) == 1
    assert kcall(row0=-1) == 1
    assert kcall(row0=600) == 1                                   # rows past N
    assert kcall(o=ops.OP_SILU_MUL) == 1                          # not with SiLU-mul
    assert kcall(n=3) == 2                                        # decode only
    assert kcall(kc=C + 8) == 3 and kcall(pos=C + 128 * MB + 2) == 3
    assert kcall(kc=A + 24 * MB) == 4                             # cache over y
    assert kcall(vc=C) == 4                                       # v cache over k cache


def fused_plan_soundness(L):
    R = ops.OP_RMSNORM_X
    for n_max in (1, 3, 17, 300):
        nb = ops.plan_workspace_fused(n_max, 4096, 11008, R)
        for n in range(1, n_max + 1, max(1, n_max // 7)):
            assert fcall(L, ops_=R, n=n, K=4096, N=11008, w=A + 64 * MB, s=A + 128 * MB, y=A + 256 * MB,
                         gamma=A + 512 * MB, ws=A + 1024 * MB, wsb=nb) == 6


def repack_validation(L):
    P = A + 64 * MB
    assert L.relax_q4_repack(A, A + MB, 256, 64, 3, 32, P, P + MB, None) == 1      # unknown layout
    assert L.relax_q4_repack(A, A + MB, 256, 64, 2, 32, P, P + MB, None) == 6      # 3-bit NK: valid
    assert L.relax_q4_repack(A, A + MB, 256, 64, 1, 48, P, P + MB, None) == 2      # group not 32/64/128
    assert L.relax_q4_repack(A, A + MB, 320, 64, 1, 128, P, P + MB, None) == 2     # K % G != 0
    assert L.relax_q4_repack(A, A + MB, 256, 64, 1, 64, 0, P + MB, None) == 1
    assert L.relax_q4_repack(A + 4, A + MB, 256, 64, 1, 64, P, P + MB, None) == 3
    assert L.relax_q4_repack(A, A + MB, 256, 64, 1, 64, A, P + MB, None) == 4      # output over the input
    assert L.relax_q4_repack(A, A + MB, 256, 0, 1, 64, P, P + MB, None) == 0       # N == 0: no-op
    assert L.relax_q4_repack(A, A + MB, 256, 64, 1, 64, P, P + MB, None) == 6      # valid: device check


def allreduce_validation(L):
    """relax_q4_matmul_allreduce (F1) and relax_tp_comm_bytes."""
    nb = ctypes.c_size_t(0)
    assert L.relax_tp_comm_bytes(0, 4096, ctypes.byref(nb)) == 1
    assert L.relax_tp_comm_bytes(9, 4096, ctypes.byref(nb)) == 1
    assert L.relax_tp_comm_bytes(2, 0, ctypes.byref(nb)) == 1
    assert L.relax_tp_comm_bytes(2, 4096, None) == 1
    assert L.relax_tp_comm_bytes(2, 4096, ctypes.byref(nb)) == 0
    # epoch counters, then 2 parities x world x 2 tokens x N (epoch, fp32) words
    assert nb.value == 1024 * 4 + 2 * 2 * 2 * 4096 * 8
    B = A + 128 * MB

    def comm(world=2, rank=0, bufs=None, nbytes=None):
        c = ops.TpComm()
        c.world, c.rank = world, rank
        for p, b in enumerate(bufs if bufs is not None else [B + p * 4 * MB for p in range(world)]):
            c.bufs[p] = b
        L.relax_tp_comm_bytes(max(1, min(world, 8)), 256, ctypes.byref(nb))
        c.buf_bytes = nb.value if nbytes is None else nbytes
        return c

    def ar(c, x=A, n=1, K=256, N=256, w=A + 8 * MB, s=A + 16 * MB, res=0, y=A + 24 * MB):
        return L.relax_q4_matmul_allreduce(ctypes.byref(c) if c is not None else None, x, n, K, N, w, s, res, y,
                                           None)
    assert ar(None) == 1
    assert ar(comm(world=0)) == 1
    assert ar(comm(world=9, bufs=[B] * 8)) == 1
    assert ar(comm(rank=2)) == 1
    assert ar(comm(bufs=[B, 0])) == 1                   # a missing peer buffer
    assert ar(comm(bufs=[B, B + 4 * MB + 8])) == 3       # misaligned peer buffer
    assert ar(comm(nbytes=1024)) == 5                    # buffer too small for N
    assert ar(comm(), n=-1) == 1
    assert ar(comm(), K=100) == 2
    assert ar(comm(), n=3) == 2                          # decode only (n <= 2)
    assert ar(comm(), K=288) == 2                        # K % 256 != 0
    assert ar(comm(), n=0, x=0, y=0) == 0                # no-op
    assert ar(comm(), y=0) == 1
    assert ar(comm(), x=A + 2) == 3
    assert ar(comm(), y=A + 8 * MB) == 4                 # y over the weights
    assert ar(comm(), y=B) == 4                          # y over this rank's exchange buffer
    assert ar(comm(), res=A + 24 * MB + 16) == 4         # partial overlap with residual
    assert ar(comm(), res=A + 24 * MB) == 6              # in-place residual is allowed
    assert ar(comm()) == 6                               # valid: device check
    assert ar(comm(world=1, bufs=[B])) == 6


def chain_validation(L):
    """relax_q4_chain_* (the persistent decode chain)."""
    nb = ctypes.c_size_t(0)
    assert L.relax_q4_chain_workspace(0, ctypes.byref(nb)) == 1
    assert L.relax_q4_chain_workspace(3, None) == 1
    assert L.relax_q4_chain_workspace(3, ctypes.byref(nb)) == 0 and nb.value > 0
    W = A + 256 * MB

    def op(x=A, w=A + 8 * MB, s=A + 16 * MB, y=A + 24 * MB, K=4096, N=4096, after=0, reserved=0):
        return ops.ChainOp(x, w, s, y, K, N, after, reserved)

    def init(oplist, ws=W, wsb=None):
        arr = (ops.ChainOp * len(oplist))(*oplist)
        return L.relax_q4_chain_init(arr, len(oplist), ws, nb.value if wsb is None else wsb)
    L.relax_q4_chain_workspace(2, ctypes.byref(nb))
    assert L.relax_q4_chain_init(None, 2, W, nb.value) == 1
    assert init([op(), op(x=0)]) == 1
    assert init([op(), op(reserved=1)]) == 1
    assert init([op(), op(K=0)]) == 1
    assert init([op(), op(K=4128)]) == 2                 # K % 256 != 0
    assert init([op(), op(K=32768)]) == 2                # more than 30 K-column warps
    assert init([op(), op(x=A + 2)]) == 3
    assert init([op(), op(y=A + 8 * MB)]) == 4           # y over the weights
    assert init([op(), op(y=A)]) == 4                    # y over its own x
    assert init([op(), op()], wsb=16) == 5
    assert init([op(), op()], ws=0) == 1
    assert init([op(), op(x=A + 24 * MB, y=A + 32 * MB, after=1)]) == 6   # x = the previous y: valid
    assert L.relax_q4_chain_run(None, None) == 1
    assert L.relax_q4_chain_run(W, None) == 6


def main():
    assert os.environ.get("CUDA_VISIBLE_DEVICES", None) == "", "run with CUDA_VISIBLE_DEVICES=''"
    L = ops.lib()
    for f in (validation_codes, workspace_too_small, plan_invalid, fused_validation_codes, fused_plan_soundness,
              repack_validation, allreduce_validation, kv_append_validation):
        f(L)
        print("ok", f.__name__)
    if hasattr(L, "relax_q4_chain_run"):            # the experiments build (RELAX_Q4_LIB)
        chain_validation(L)
        print("ok chain_validation")
    print("ALL OK")


if __name__ == "__main__":
    main()
