"""GPU parity of the row split with its all-reduce fused into the decode kernel
(relax_q4_matmul_allreduce; include/relax_q4.h; DESIGN.md
§8.1), against the fp64 oracle of the full-K matmul: the row split only
re-associates the K sum, y = sum_p x_p . W_p = x . W (P:471-494 fuse the
consumer -- here the sum -- into the producer).

Two settings, both on one GPU and neither with kernels waiting on each other:
  * NCCL world size 1 through tp.TpExchange (torch symmetric memory): the
    product set-up and the per-CTA epoch counters (the rank's own partial is
    summed from registers, so no words move); eager, repeated and captured in
    a CUDA graph.
  * emulated peers: world 2..8, this process is rank r and the other ranks'
    contributions are placed in its exchange buffer beforehand -- their fp32
    partials from the ORACLE (x_p . W_p of their K slices) in (epoch, value)
    words of the call's epoch -- so the kernel finds every peer already
    arrived.  The words this rank stores into the "peer" buffers (plain device
    allocations) are checked too.  This covers offsets, the world > 1 slot
    layout and the sum order without a second GPU."""
import ctypes
import os
import socket

import numpy as np
import pytest

import oracle
from oracle import fused as ofu
from paper_2311_02103_b200 import inputs, ops, tp
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HDR_BYTES = 1024 * 4                      # epoch counters (csrc/internal.h kTp*), then the words


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


SHAPES = [(1024, 8192), (3584, 8192), (512, 4096), (256, 1000), (4096, 4096)]   # 70B o / down at TP8, 7B o at TP8


@pytest.mark.parametrize("n", [1, 2])
def test_world1_matches_plain_and_oracle(nccl_group, n):
    """At world 1 the fused sum is the rank's own fp32 partial: bitwise the
    plain decode kernel's output, and within tolerance of the oracle; with the
    residual, bitwise the plain fused-residual kernel."""
    ex = tp.TpExchange(8192, group=nccl_group)
    for i, (K, N) in enumerate(SHAPES):
        pk, sc = inputs.realistic_weights(8100 + i, K, N)
        w = dev_weights(pk, sc)
        x = inputs.activations(8200 + i + n, n, K)
        res = inputs.activations(8300 + i + n, n, N)
        xd, rd = dev_x(x), dev_x(res)
        y = ops.q4_matmul_allreduce(xd, *w, ex.comm)
        yr = ops.q4_matmul_allreduce(xd, *w, ex.comm, residual=rd)
        plain = ops.q4_matmul(xd, *w)
        plain_r = ops.q4_matmul_fused(xd, *w, residual=rd)
        torch.cuda.synchronize()
        r = oracle.matmul_f64(x, pk, sc, K, N)
        assert_within_tol(host_bits(y), r, f"allreduce world1 K={K} N={N} n={n}")
        assert np.array_equal(host_bits(y), host_bits(plain)), (K, N, n)
        assert np.array_equal(host_bits(yr), host_bits(plain_r)), (K, N, n)
        got = host_bits(yr).view(np.float16).astype(np.float64)
        want = ofu.residual(r, res)
        rel = np.abs(got - want) / np.maximum(np.abs(want), np.sqrt(np.mean(want * want)))
        assert rel.max() <= 1e-2, rel.max()
    # every CTA of every call advanced its epoch counter by one per call
    hdr = ex.buf[:4 * 1024].view(torch.int32).cpu().numpy()
    grid = max(int(np.count_nonzero(hdr)), 1)
    assert set(np.unique(hdr[:grid]).tolist()) <= {2 * len(SHAPES)}, np.unique(hdr)


def test_world1_repeated_and_graph(nccl_group):
    """Many calls (alternating partial slots, epochs climbing) interleaved with
    other kernels, then the same sequence captured in a CUDA graph and
    replayed: every output equals the first eager result bit for bit."""
    ex = tp.TpExchange(8192, group=nccl_group)
    mats = [inputs.realistic_weights(8400 + i, K, N) for i, (K, N) in enumerate(SHAPES[:3])]
    dw = [dev_weights(*m) for m in mats]
    xs = [dev_x(inputs.activations(8500 + i, 1, K)) for i, (K, _) in enumerate(SHAPES[:3])]
    ys = [torch.empty((1, N), dtype=torch.float16, device="cuda") for _, N in SHAPES[:3]]
    st = torch.cuda.Stream()

    def seq():
        for x, w, y in zip(xs, dw, ys):
            ops.q4_matmul_allreduce(x, *w, ex.comm, y=y, stream=st)
            ops.q4_matmul(x, *w, stream=st)          # an unrelated kernel between fused calls

    with torch.cuda.stream(st):
        seq()
    torch.cuda.synchronize()
    first = [host_bits(y) for y in ys]
    for (K, N), (pk, sc), x, y in zip(SHAPES[:3], mats, xs, first):
        assert_within_tol(y, oracle.matmul_f64(host_bits(x), pk, sc, K, N), f"allreduce K={K}")
    for _ in range(5):
        with torch.cuda.stream(st):
            seq()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        seq()
    for _ in range(7):
        for y in ys:
            y.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for y, f in zip(ys, first):
            assert np.array_equal(host_bits(y), f)


def test_row_parallel_uses_fused_path(nccl_group):
    """tp.RowParallelQ4 with an exchange: decode goes through the fused call
    (same bits as calling it directly), larger n through matmul + NCCL."""
    ex = tp.TpExchange(4096, group=nccl_group)
    K, N = 1024, 4096
    pk, sc = inputs.realistic_weights(8600, K, N)
    w = dev_weights(pk, sc)
    lin = tp.megatron_linear("o", *w, group=nccl_group, exchange=ex)
    for n in (1, 2, 5):
        x = inputs.activations(8610 + n, n, K)
        y = host_bits(lin(dev_x(x)))
        torch.cuda.synchronize()
        assert_within_tol(y, oracle.matmul_f64(x, pk, sc, K, N), f"RowParallelQ4 exchange n={n}")
        if n <= 2:
            assert np.array_equal(y, host_bits(ops.q4_matmul_allreduce(dev_x(x), *w, ex.comm)))


def _slot_off(parity, src, t, row, world, N):
    return HDR_BYTES + ((((parity * world + src) * 2 + t) * N) + row) * 8


def _words(values_f32, epoch):
    """(epoch << 32) | fp32 bits, little-endian u64 words."""
    v = np.ascontiguousarray(values_f32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return (v | (np.uint64(epoch) << np.uint64(32))).view(np.uint8)


@pytest.mark.parametrize("world,rank", [(2, 0), (2, 1), (4, 3), (8, 5)])
@pytest.mark.parametrize("n", [1, 2])
def test_emulated_peers(world, rank, n):
    """World > 1 on one GPU: the other ranks' partials (oracle fp32 of their K
    slices, as words of epoch 1) sit in this rank's buffer before the call; y
    must be the oracle of the full-K matmul, and the words this rank stored
    into each peer buffer must be its own slice's partial with epoch 1."""
    Kp, N = 512, 1000
    K = Kp * world
    pk, sc = inputs.realistic_weights(8700 + world + rank, K, N)
    x = inputs.activations(8800 + world + rank + n, n, K)
    shards = [tp.shard_rows(pk, sc, p, world) for p in range(world)]
    xsl = [tp.split_x_for_rows(x, p, world) for p in range(world)]
    nbytes = ops.tp_comm_bytes(world, N)
    bufs = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
    own = np.zeros(nbytes, dtype=np.uint8)
    e = 1                                                    # the first call's epoch
    parts = {}
    for p in range(world):
        parts[p] = oracle.matmul_f64(xsl[p], *shards[p], Kp, N).astype(np.float32)   # [n][N]
        if p == rank:
            continue
        for t in range(n):
            o = _slot_off(e & 1, p, t, 0, world, N)
            own[o:o + 8 * N] = _words(parts[p][t], e)
    bufs[rank].copy_(torch.from_numpy(own))
    comm = ops.make_tp_comm(world, rank, [b.data_ptr() for b in bufs], nbytes)
    w = dev_weights(*shards[rank])
    y = ops.q4_matmul_allreduce(dev_x(xsl[rank]), *w, comm)
    torch.cuda.synchronize()
    r = oracle.matmul_f64(x, pk, sc, K, N)
    assert_within_tol(host_bits(y), r, f"emulated world={world} rank={rank} n={n}")
    # the words this rank stored: slot (parity 1, src rank) of every other buffer
    mine = None
    for p in range(world):
        if p == rank:
            continue
        b = bufs[p].cpu().numpy()
        got = []
        for t in range(n):
            o = _slot_off(e & 1, rank, t, 0, world, N)
            wd = b[o:o + 8 * N].view(np.uint64)
            assert np.all((wd >> np.uint64(32)) == e), (p, t)
            got.append((wd & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32))
            ref = parts[rank][t].astype(np.float64)
            d = np.abs(got[-1].astype(np.float64) - ref)
            assert d.max() <= 1e-3 * np.sqrt(np.mean(ref * ref)) + 1e-6, (p, t)
        got = np.stack(got)
        if mine is not None:
            assert np.array_equal(got.view(np.uint32), mine.view(np.uint32))   # the same words to every peer
        mine = got
        # nothing else was written into the peer's buffer: its counters stay 0
        assert not b[:HDR_BYTES].any()
    # this rank's own epoch counters: one call on its grid of CTAs
    ctr = bufs[rank][:HDR_BYTES].view(torch.int32).cpu().numpy()
    grid = int(np.count_nonzero(ctr))
    assert grid >= 1 and np.all(ctr[:grid] == e) and np.all(ctr[grid:] == 0)
    # the sum is taken in rank order: y == fp16(sum_p partial_p) exactly, the
    # own partial being the one it sent (mine), the others the placed words
    acc = None
    for p in range(world):
        v = mine if p == rank else parts[p][:n]
        acc = v.copy() if acc is None else acc + v
    assert np.array_equal(host_bits(y), acc.astype(np.float16).view(np.uint16))
