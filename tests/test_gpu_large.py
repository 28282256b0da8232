"""Very wide outputs on the GPU (advisor r1: a 405B-class lm_head, 128k-256k
vocabularies): the decode dispatch must pick a schedule whose shared-memory
footprint fits for the real N, and the result must match the oracle.  The
weights are random device tensors (any 32-bit word is a valid q4 code word);
the sampled output columns are checked against the oracle on the same rows
copied back to the host."""
import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("K,N", [(16384, 128256), (8192, 256000)])
@pytest.mark.parametrize("n", [1, 2, 5])
def test_wide_lm_head(K, N, n):
    g = torch.Generator(device="cuda")
    g.manual_seed(K + N)
    pk = torch.randint(-2 ** 31, 2 ** 31 - 1, (N, K // 8), dtype=torch.int32, device="cuda", generator=g)
    # scales: small positive fp16 (2^-10 .. 2^-6)
    sc = (torch.rand((N, K // 32), device="cuda", generator=g) * (2 ** -6 - 2 ** -10) + 2 ** -10).half()
    x = inputs.activations(900 + n, n, K)
    y = host_bits(ops.q4_matmul(dev_x(x), pk, sc, ws=ops.workspace(n, K, N)))
    torch.cuda.synchronize()
    rng = np.random.default_rng(n)
    cols = np.unique(np.concatenate([[0, N - 1], rng.choice(N, 24, replace=False)]))
    idx = torch.from_numpy(cols).cuda()
    pk_h = pk.index_select(0, idx).cpu().numpy().view(np.uint32)
    sc_h = sc.index_select(0, idx).cpu().numpy().view(np.uint16)
    r = oracle.matmul_f64(x, pk_h, sc_h, K, len(cols))
    assert_within_tol(y[:, cols], r, f"wide {K}x{N} n={n} sched={ops.query_schedule(n, K, N)}")
