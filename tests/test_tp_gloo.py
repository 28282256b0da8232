"""Tensor-parallel host logic on CPU: world_size 2 over gloo (127.0.0.1).

The per-rank matmul here is the CPU oracle (test-only injection); on the GPU
box the same classes call the C-ABI kernel.  Checks (SURVEY §8(c) "TP"):
column shards concatenated == the unsharded oracle bitwise (columns are
independent); row-split partial sums all-reduced == unsharded oracle within
tolerance; the Megatron pair (column -> row) matches the two-step oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2311_02103_b200 import inputs, tp
from tests._util import assert_within_tol


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_mm(x, pk, sc):
    xb = x.contiguous().numpy().view(np.uint16)
    pkn = pk.contiguous().numpy().view(np.uint32)
    scn = sc.contiguous().numpy().view(np.uint16)
    K = xb.shape[1]
    N = pkn.shape[0]
    r = oracle.matmul_f64(xb, pkn, scn, K, N, nthreads=1)
    return torch.from_numpy(oracle.round_f16(r).view(np.float16).copy())


def t16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.float16).copy())


def t32(words):
    return torch.from_numpy(np.ascontiguousarray(words).view(np.int32).copy())


def _worker(rank, world, port, q):
    try:
        _worker_body(rank, world, port, q)
    except BaseException as e:  # noqa: BLE001  -- fail the test now, not at the queue timeout
        q.put((rank, {"error": repr(e)}))
        raise


def _worker_body(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        K, N, n = 512, 256, 3
        pk, sc = inputs.realistic_weights(5000, K, N)
        xb = inputs.activations(5001, n, K)
        x = t16(xb)
        # column split + all_gather
        cpk, csc = tp.shard_columns(t32(pk), t16(sc), rank, world)
        col = tp.ColumnParallelQ4(cpk, csc, gather=True, matmul=oracle_mm)
        out["col"] = col(x).numpy().view(np.uint16)
        # row split + all_reduce
        rpk, rsc = tp.shard_rows(t32(pk), t16(sc), rank, world)
        row = tp.RowParallelQ4(rpk, rsc, matmul=oracle_mm)
        out["row"] = row(tp.split_x_for_rows(x, rank, world)).numpy().view(np.uint16)
        # Megatron pair: gate (col, K->N2) then down (row, N2->K2)
        K2 = 256
        gpk, gsc = inputs.realistic_weights(5002, K, 512)          # K -> 512
        dpk, dsc = inputs.realistic_weights(5003, 512, K2)         # 512 -> K2
        g = tp.ColumnParallelQ4(*tp.shard_columns(t32(gpk), t16(gsc), rank, world), matmul=oracle_mm)
        d = tp.RowParallelQ4(*tp.shard_rows(t32(dpk), t16(dsc), rank, world), matmul=oracle_mm)
        out["pair"] = d(g(x)).numpy().view(np.uint16)
        # lm_head: column split, logits all-gathered (all_gather_into_tensor) back
        # into feature order for n = 3 tokens
        hpk, hsc = inputs.realistic_weights(5004, K, 320)
        head = tp.megatron_linear("lm_head", *tp.shard_columns(t32(hpk), t16(hsc), rank, world), matmul=oracle_mm)
        out["head"] = head(x).numpy().view(np.uint16)
        # the shard shapes the bench uses agree with the shards themselves
        out["shapes"] = [tuple(tp.shard_columns(t32(hpk), t16(hsc), rank, world)[0].shape),
                         tp.shard_shape("lm_head", K, 320, world), tp.shard_shape("down", 512, K2, world)]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    oracle.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for r, out in res.items():
        assert "error" not in out, f"rank {r}: {out['error']}"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_column_split_bitwise(results):
    K, N, n = 512, 256, 3
    pk, sc = inputs.realistic_weights(5000, K, N)
    xb = inputs.activations(5001, n, K)
    want = oracle.round_f16(oracle.matmul_f64(xb, pk, sc, K, N))
    for r in (0, 1):
        assert np.array_equal(results[r]["col"], want)


def test_row_split_allreduce_within_tol(results):
    K, N, n = 512, 256, 3
    pk, sc = inputs.realistic_weights(5000, K, N)
    xb = inputs.activations(5001, n, K)
    r = oracle.matmul_f64(xb, pk, sc, K, N)
    assert np.array_equal(results[0]["row"], results[1]["row"])
    assert_within_tol(results[0]["row"], r, "row split")


def test_megatron_pair(results):
    K, n = 512, 3
    xb = inputs.activations(5001, n, K)
    gpk, gsc = inputs.realistic_weights(5002, K, 512)
    dpk, dsc = inputs.realistic_weights(5003, 512, 256)
    h = oracle.round_f16(oracle.matmul_f64(xb, gpk, gsc, K, 512))
    r = oracle.matmul_f64(h, dpk, dsc, 512, 256)
    assert np.array_equal(results[0]["pair"], results[1]["pair"])
    assert_within_tol(results[0]["pair"], r, "pair")


def test_lm_head_gather_feature_order(results):
    """Column-split logits, all-gathered: identical on both ranks and equal,
    bitwise, to the unsharded oracle for n > 1 (the [p][n][N/p] gather buffer is
    reordered to [n][N])."""
    K, n = 512, 3
    xb = inputs.activations(5001, n, K)
    hpk, hsc = inputs.realistic_weights(5004, K, 320)
    want = oracle.round_f16(oracle.matmul_f64(xb, hpk, hsc, K, 320))
    for r in (0, 1):
        assert results[r]["head"].shape == (n, 320)
        assert np.array_equal(results[r]["head"], want)
    assert results[0]["shapes"][0] == (160, 512 // 8)
    assert results[0]["shapes"][1] == (512, 160)
    assert results[0]["shapes"][2] == (256, 256)


def test_shard_bounds_errors():
    with pytest.raises(ValueError):
        tp.shard_bounds(100, 0, 3)
    with pytest.raises(ValueError):
        tp.shard_bounds(96, 0, 2, align=32)   # 48 not a multiple of 32
    assert tp.shard_bounds(8192, 3, 8, 32) == (3072, 4096)


def test_fused_allreduce_routing():
    """Which row-split calls take the fused decode all-reduce (include/relax_q4.h
    relax_q4_matmul_allreduce: n <= 2, K % 256 == 0): the Llama TP shards of o
    and down, and the ones that fall back to matmul + NCCL."""
    assert tp.fused_allreduce_ok(1, 1024) and tp.fused_allreduce_ok(2, 3584)      # 70B o / down at TP8
    assert tp.fused_allreduce_ok(1, 512)                                           # 7B o at TP8
    assert not tp.fused_allreduce_ok(1, 1376)                                      # 7B down at TP8 (11008 / 8)
    assert not tp.fused_allreduce_ok(3, 1024) and not tp.fused_allreduce_ok(0, 1024)
    K, N = tp.shard_shape("down", 28672, 8192, 8)
    assert (K, N) == (3584, 8192) and tp.fused_allreduce_ok(1, K)
    # without an exchange RowParallelQ4 never takes the fused path (CPU, gloo-testable)
    lin = tp.RowParallelQ4(None, None, matmul=lambda x, pk, sc: x)
    assert lin.exchange is None
