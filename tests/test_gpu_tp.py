"""The tensor-parallel data path (paper_2311_02103_b200/tp.py) on the GPU over
NCCL, world size 1 (the only size one B200 box offers; N > 1 is covered by the
gloo tests on CPU).  The same code path runs at every world size -- the NCCL
all_gather_into_tensor / all_reduce are executed, not short-cut -- with the
product kernel as the per-rank matmul, eagerly and captured in a CUDA graph
(as bench.py times it), against the fp64 oracle (SURVEY §8(c) "TP")."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops, tp
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


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


@pytest.mark.parametrize("n", [1, 3, 64, 300])
def test_megatron_layer_world1(nccl_group, n):
    """qkv (column) -> o (row, all_reduce fp32) and gate_up (column) -> down
    (row), lm_head (column, logits all-gathered); each output against the
    oracle on sampled columns."""
    cases = [("qkv", 1024, 1536), ("o", 1024, 1024), ("gate_up", 1024, 2816), ("down", 1408, 1024),
             ("lm_head", 1024, 4000)]
    st = torch.cuda.Stream()
    mm = lambda x, pk, sc: ops.q4_matmul(x, pk, sc, stream=st)   # noqa: E731
    host, lin, xs = [], [], []
    for i, (name, K, N) in enumerate(cases):
        pk, sc = inputs.realistic_weights(9900 + i, K, N)
        host.append((pk, sc))
        lin.append(tp.megatron_linear(name, *dev_weights(pk, sc), group=nccl_group, matmul=mm))
        xs.append(inputs.activations(9950 + i + n, n, K))
    xd = [dev_x(x) for x in xs]
    with torch.cuda.stream(st):
        eager = [host_bits(f(x)) for f, x in zip(lin, xd)]
    torch.cuda.synchronize()
    rng = np.random.default_rng(n)
    for (name, K, N), (pk, sc), x, y in zip(cases, host, xs, eager):
        assert y.shape == (n, N), (name, y.shape)
        cols = np.unique(np.concatenate([[0, N - 1], rng.choice(N, 40, replace=False)]))
        r = oracle.matmul_cols_f64(x, pk, sc, K, cols)
        assert_within_tol(y[:, cols], r, f"tp world1 {name} n={n}")
    # the bench's launch configuration: the whole set, collectives included, in one CUDA graph
    outs = [None] * len(lin)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i, (f, x) in enumerate(zip(lin, xd)):
            outs[i] = f(x)
    g.replay()
    torch.cuda.synchronize()
    for e, o in zip(eager, outs):
        assert np.array_equal(e, host_bits(o))
