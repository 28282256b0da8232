"""GPU parity of relax_q4_matmul_grouped (several linears reading the same x in
one decode launch): every member against the fp64 oracle, the pinned cases
bitwise, in the benchmark's CUDA-graph chain."""
import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GROUPS = {
    "qkv7b": [(4096, 4096)] * 3,
    "gate_up7b": [(4096, 11008)] * 2,
    "qkv70b_gqa": [(8192, 8192), (8192, 1024), (8192, 1024)],
    "ragged": [(768, 328), (768, 40), (768, 1000), (768, 8)],
}


@pytest.mark.parametrize("name", list(GROUPS))
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 17])
def test_grouped_members_match_oracle(name, n):
    mats = GROUPS[name]
    K = mats[0][0]
    host = [inputs.realistic_weights(7000 + i + n, K, N) for i, (_, N) in enumerate(mats)]
    devw = [dev_weights(p, s) for p, s in host]
    x = inputs.activations(7100 + n, n, K)
    ys = ops.q4_matmul_grouped(dev_x(x), devw)
    torch.cuda.synchronize()
    rng = np.random.default_rng(n)
    for i, ((_, N), (pk, sc), y) in enumerate(zip(mats, host, ys)):
        cols = np.unique(np.concatenate([[0, N - 1], rng.choice(N, min(N, 40), replace=False)]))
        r = oracle.matmul_cols_f64(x, pk, sc, K, cols)
        assert_within_tol(host_bits(y)[:, cols], r, f"grouped {name} member {i} n={n}")


def test_grouped_smalln_equals_single_calls():
    """3 <= n <= 8: one small-batch launch for the group; each member equals
    the member's own relax_q4_matmul (the same kernel over the same rows,
    another CTA split) bit for bit."""
    K = 4096
    for mats in (GROUPS["qkv7b"], GROUPS["gate_up7b"], GROUPS["qkv70b_gqa"][:1] + [(4096, 1024), (4096, 1024)]):
        host = [inputs.realistic_weights(7400 + i, K, N) for i, (_, N) in enumerate(mats)]
        devw = [dev_weights(p, s) for p, s in host]
        for n in (3, 8):
            x = dev_x(inputs.activations(7500 + n, n, K))
            ys = ops.q4_matmul_grouped(x, devw)
            for (pk, sc), y in zip(devw, ys):
                single = ops.q4_matmul_ex(x, pk, sc, variant=ops.VARIANT_SMALLN)
                assert np.array_equal(host_bits(y), host_bits(single))


def test_grouped_pinned_cases_bitwise():
    """One-hot rows extract W and all-7 members give exact zeros, as for single calls."""
    K = 512
    mats = [(K, 256), (K, 64), (K, 130)]
    host = [inputs.stress_weights(7200 + i, K, N) for i, (_, N) in enumerate(mats)]
    host[1] = (np.full_like(host[1][0], 0x77777777), host[1][1])
    devw = [dev_weights(p, s) for p, s in host]
    for n, ks in ((1, [5]), (2, [0, 511]), (4, [0, 7, 300, 511])):
        x = np.zeros((n, K), dtype=np.uint16)
        for i, k in enumerate(ks):
            x[i, k] = 0x3C00
        ys = ops.q4_matmul_grouped(dev_x(x), devw)
        torch.cuda.synchronize()
        for j, ((pk, sc), (_, N), y) in enumerate(zip(host, mats, ys)):
            W = oracle.dequant(pk, sc, K, N)
            got = host_bits(y)
            for i, k in enumerate(ks):
                if j == 1:                                   # codes all 7: W == 0, y == +-0
                    assert np.all(got[i] & 0x7FFF == 0)
                else:
                    assert np.array_equal(got[i], W[:, k]), (j, n, k)


def test_grouped_in_graph_chain():
    """The bench's configuration: grouped q/k/v then a dependent o, captured in
    a CUDA graph with PDL, replayed; each stage against the oracle of the
    previous stage's GPU output."""
    K = 1024
    qkv = [inputs.realistic_weights(7300 + i, K, K) for i in range(3)]
    o = inputs.realistic_weights(7310, K, K)
    dq = [dev_weights(p, s) for p, s in qkv]
    do = dev_weights(*o)
    x0 = inputs.activations(7320, 1, K)
    x = dev_x(x0)
    ys = [torch.empty((1, K), dtype=torch.float16, device="cuda") for _ in range(3)]
    yo = torch.empty((1, K), dtype=torch.float16, device="cuda")
    st = torch.cuda.Stream()

    def chain():
        ops.q4_matmul_grouped(x, dq, ys=ys, stream=st)
        ops.q4_matmul(ys[2], do[0], do[1], y=yo, stream=st)

    with torch.cuda.stream(st):
        chain()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        chain()
    for y in ys + [yo]:
        y.fill_(float("nan"))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for (pk, sc), y in zip(qkv, ys):
        assert_within_tol(host_bits(y), oracle.matmul_f64(x0, pk, sc, K, K), "grouped member in chain")
    v = host_bits(ys[2])
    assert_within_tol(host_bits(yo), oracle.matmul_f64(v, *o, K, K), "dependent o after the group")
