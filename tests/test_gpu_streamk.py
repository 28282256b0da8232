"""GPU parity of the stream-K schedule of the persistent tensor-core kernel
(relax_query_schedule persistent == 2): the full waves of
pair tiles run whole, the rest tiles are cut into (tile, 256-k stage) units
spread evenly over the CTA pairs and run first, tiles cut between pairs
reduced through the workspace by the pair that completes them, in fixed pair
order (experiments build with RELAX_Q4_STREAMK=1: measured slower than the
product's schedules).

Against the fp64 oracle on sampled columns (every token row; the first and
last columns and those of the cut tiles always), rerun bitwise
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

# (K, N, n): 4096 x 11008 / 12288 at n = 300 / 512 (one full wave + rest),
# 4096^2 and 11008 x 4096 at n = 2048 (k = 16 / 43 stages), a ragged N and n,
# the 7B lm_head at n = 512 (three full waves + rest)
CASES = [(4096, 11008, 512), (4096, 12288, 300), (4096, 4096, 2048), (11008, 4096, 2048), (4096, 11008, 777),
         (2048, 2000, 3000), (4096, 32000, 512)]


@pytest.mark.parametrize("K,N,n", CASES)
def test_stream_k_matches_oracle(K, N, n):
    q = ops.query_schedule(n, K, N)
    assert q.get("stream_k"), q
    pk, sc = inputs.realistic_weights(5300 + K + N + n, K, N)
    w = dev_weights(pk, sc)
    x = inputs.activations(5400 + n, n, K)
    xd = dev_x(x)
    ws = torch.zeros(max(ops.plan_workspace(n, K, N), q["ws_bytes"]), dtype=torch.uint8, device="cuda")
    y = host_bits(ops.q4_matmul(xd, *w, ws=ws))
    torch.cuda.synchronize()
    assert not ws[:4096].any(), "ticket region not zero after the call"
    rng = np.random.default_rng(n)
    # the cut tiles are the last pair tiles (m-tile pairs fastest, 256 rows x 256 tokens each)
    cols = np.unique(np.concatenate([[0, N - 1], rng.choice(N, 48, replace=False),
                                     np.arange(max(0, N - 3072), N, 23)]))
    r = oracle.matmul_cols_f64(x, pk, sc, K, cols)
    assert_within_tol(y[:, cols], r, f"stream-K {K}x{N} n={n} sched={q}")
    again = host_bits(ops.q4_matmul(xd, *w, ws=ws))
    assert np.array_equal(y, again)
    # without a workspace the call takes a workspace-free schedule (same tolerance)
    y2 = host_bits(ops.q4_matmul(xd, *w))
    assert_within_tol(y2[:, cols], r, f"no-workspace fallback {K}x{N} n={n}")


def test_stream_k_is_chosen_for_quantised_grids():
    """The dispatch offers stream-K where whole tiles quantise badly (172
    single tiles on 148 SMs), and not where they fill the waves."""
    assert ops.query_schedule(512, 4096, 11008).get("stream_k")
    assert not ops.query_schedule(4096, 4096, 11008).get("stream_k")
    assert not ops.query_schedule(512, 4096, 4096).get("stream_k")
