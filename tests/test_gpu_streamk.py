"""GPU parity of the stream-K schedule of the persistent tensor-core kernel
(relax_query_schedule persistent == 2; experiments build with
RELAX_Q4_STREAMK=1, measured slower than the product's schedules): the (tile, 256-k
stage) units spread evenly over the CTA pairs, tiles cut between pairs reduced
through the workspace by the pair that completes them, in fixed pair order.

Against the fp64 oracle on sampled columns (every token row), rerun bitwise
(deterministic), the ticket region of the workspace zero again after every
call, and a relax_q4_matmul call without workspace falling back to another
schedule with the same tolerance."""
import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ops.query_schedule(512, 4096, 11008).get("stream_k"),
                                 reason="stream-K is offered only by the experiments build with RELAX_Q4_STREAMK=1 "
                                        "(measured slower, DESIGN.md §5.8; tools/gpu_streamk.sh)")]

torch = pytest.importorskip("torch")

CASES = [(4096, 11008, 512), (4096, 12288, 256), (4096, 4096, 2048), (11008, 4096, 2048), (4096, 11008, 300),
         (2048, 2000, 777)]


@pytest.mark.parametrize("K,N,n", CASES)
def test_stream_k_matches_oracle(K, N, n):
    q = ops.query_schedule(n, K, N)
    pk, sc = inputs.realistic_weights(5300 + K + N + n, K, N)
    w = dev_weights(pk, sc)
    x = inputs.activations(5400 + n, n, K)
    xd = dev_x(x)
    ws = torch.zeros(max(ops.plan_workspace(n, K, N), q["ws_bytes"]), dtype=torch.uint8, device="cuda")
    y = host_bits(ops.q4_matmul(xd, *w, ws=ws))
    torch.cuda.synchronize()
    assert not ws[:4096].any(), "ticket region not zero after the call"
    rng = np.random.default_rng(n)
    cols = np.unique(np.concatenate([[0, N - 1], rng.choice(N, 48, replace=False)]))
    r = oracle.matmul_cols_f64(x, pk, sc, K, cols)
    assert_within_tol(y[:, cols], r, f"stream-K {K}x{N} n={n} sched={q}")
    again = host_bits(ops.q4_matmul(xd, *w, ws=ws))
    assert np.array_equal(y, again)
    # without a workspace the call takes a workspace-free schedule (same tolerance)
    y2 = host_bits(ops.q4_matmul(xd, *w))
    assert_within_tol(y2[:, cols], r, f"no-workspace fallback {K}x{N} n={n}")


def test_stream_k_is_chosen_for_quantised_grids():
    """The dispatch offers stream-K where whole tiles quantise badly."""
    assert ops.query_schedule(512, 4096, 11008).get("stream_k")
