"""GPU parity of the persistent decode chain (relax_q4_chain_*, experiments build; include/relax_q4_debug.h;
DESIGN.md §5.10): a sequence of n = 1 matmuls in one launch, against the fp64
oracle.  Dependent ops read an earlier op's output; the oracle runs the same
chain itself (its own fp16-rounded intermediates, never the GPU's)."""
import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ops.has_chain(), reason="decode chain: experiments build only "
                                 "(tools/gpu_chain.sh sets RELAX_Q4_LIB=build_exp/librelax_q4_exp.so)")]

torch = pytest.importorskip("torch")

SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096), (4096, 32000), (1024, 8192), (512, 4096), (8192, 1024),
          (28672, 8192), (13824, 5120), (256, 40), (768, 300)]


def test_independent_ops_and_relaunch():
    """Every supported shape class in one chain (no dependencies), each op
    against the oracle; then relaunched eagerly and from a CUDA graph (the
    launch generation advancing): bitwise the first result every time."""
    host, dev, xs, ys = [], [], [], []
    for i, (K, N) in enumerate(SHAPES):
        pk, sc = inputs.realistic_weights(9100 + i, K, N)
        host.append((pk, sc))
        dev.append(dev_weights(pk, sc))
        xs.append(inputs.activations(9200 + i, 1, K))
        ys.append(torch.empty((1, N), dtype=torch.float16, device="cuda"))
    xd = [dev_x(x) for x in xs]
    ch = ops.DecodeChain([(x, w[0], w[1], y, False) for x, w, y in zip(xd, dev, ys)])
    st = torch.cuda.Stream()
    ch.run(stream=st)
    torch.cuda.synchronize()
    first = [host_bits(y) for y in ys]
    for (K, N), (pk, sc), x, y in zip(SHAPES, host, xs, first):
        assert_within_tol(y, oracle.matmul_f64(x, pk, sc, K, N), f"chain op {K}x{N}")
    for _ in range(3):
        ch.run(stream=st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ch.run(stream=st)
    for _ in range(4):
        for y in ys:
            y.fill_(float("nan"))
        with torch.cuda.stream(st):
            g.replay()
        torch.cuda.synchronize()
        for y, f in zip(ys, first):
            assert np.array_equal(host_bits(y), f)


@pytest.mark.parametrize("dims", [[4096, 4096, 11008, 4096, 4096], [1024, 8192, 1024, 2048, 512, 32000],
                                  [8192, 28672, 8192]])
def test_dependent_chain(dims):
    """x -> W0 -> W1 -> ... with each op reading the previous op's y (after = 1),
    against the oracle's own chain (fp16 between ops, as the kernel stores)."""
    mats = [inputs.realistic_weights(9300 + i, K, N) for i, (K, N) in enumerate(zip(dims[:-1], dims[1:]))]
    dev = [dev_weights(*m) for m in mats]
    x0 = inputs.activations(9400 + len(dims), 1, dims[0])
    bufs = [dev_x(x0)] + [torch.empty((1, N), dtype=torch.float16, device="cuda") for N in dims[1:]]
    ch = ops.DecodeChain([(bufs[i], *dev[i], bufs[i + 1], i > 0) for i in range(len(mats))])
    for rep in range(3):
        for b in bufs[1:]:
            b.fill_(float("nan"))
        ch.run()
        torch.cuda.synchronize()
        cur = x0
        for i, ((pk, sc), (K, N)) in enumerate(zip(mats, zip(dims[:-1], dims[1:]))):
            r = oracle.matmul_f64(cur, pk, sc, K, N)
            assert_within_tol(host_bits(bufs[i + 1]), r, f"chain step {i} ({K}x{N}) rep {rep}")
            cur = oracle.round_f16(r)


def test_layer_pattern_and_pinned_cases():
    """A Llama-layer-shaped chain (q, k, v read the same x; o after v; gate,
    up; down after up) where v's weights are all-7 codes (W = 0: v must be
    exactly +-0, and o, which reads v, exactly +-0 too) and the x of q/k/v is
    one-hot (q and k extract a column of W bit for bit)."""
    K, F = 1024, 2816
    shapes = {"q": (K, K), "k": (K, K), "v": (K, K), "o": (K, K), "gate": (K, F), "up": (K, F), "down": (F, K)}
    host = {nm: inputs.realistic_weights(9500 + i, *kn) for i, (nm, kn) in enumerate(shapes.items())}
    host["v"] = (np.full_like(host["v"][0], 0x77777777), host["v"][1])
    dev = {nm: dev_weights(*hw) for nm, hw in host.items()}
    x = np.zeros((1, K), dtype=np.uint16)
    x[0, 77] = 0x3C00
    xd = dev_x(x)
    y = {nm: torch.empty((1, kn[1]), dtype=torch.float16, device="cuda") for nm, kn in shapes.items()}
    xg = dev_x(inputs.activations(9600, 1, K))
    plan = [("q", xd, False), ("k", xd, False), ("v", xd, False), ("o", y["v"], True), ("gate", xg, True),
            ("up", xg, False), ("down", y["up"], True)]
    ch = ops.DecodeChain([(xx, *dev[nm], y[nm], after) for nm, xx, after in plan])
    ch.run()
    torch.cuda.synchronize()
    for nm in ("q", "k"):
        W = oracle.dequant(*host[nm], K, K)
        assert np.array_equal(host_bits(y[nm])[0], W[:, 77]), nm
    for nm in ("v", "o"):
        assert np.all(host_bits(y[nm]) & 0x7FFF == 0), nm
    xgh = host_bits(xg)
    for nm in ("gate", "up"):
        assert_within_tol(host_bits(y[nm]), oracle.matmul_f64(xgh, *host[nm], K, F), nm)
    r_up = oracle.round_f16(oracle.matmul_f64(xgh, *host["up"], K, F))
    assert_within_tol(host_bits(y["down"]), oracle.matmul_f64(r_up, *host["down"], F, K), "down after up")
