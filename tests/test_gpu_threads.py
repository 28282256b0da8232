"""The library is reentrant (include/relax_q4.h): host threads
calling it concurrently, each on its own CUDA stream, with every schedule class
(streamed decode, small-batch warp MMA, tensor-core tiles with split-K
clusters, the persistent kernel) get the same bits as one thread calling it
alone.  Python threads release the GIL inside the ctypes calls, so the C-ABI's
per-device init, kernel-attribute setup and per-thread tensor-map caches run
concurrently here."""
import threading

import numpy as np
import pytest

from paper_2311_02103_b200 import inputs, ops
from tests._util import dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = [(4096, 4096, 1), (4096, 11008, 2), (4096, 4096, 8), (1024, 2048, 48), (4096, 11008, 1024), (2048, 4096, 300)]


def test_concurrent_threads_bitwise_equal_to_serial():
    weights = [dev_weights(*inputs.realistic_weights(4400 + i, K, N)) for i, (K, N, _) in enumerate(CASES)]
    xs = [dev_x(inputs.activations(4500 + i, n, K)) for i, (K, N, n) in enumerate(CASES)]
    wss = [ops.workspace(n, K, N) for K, N, n in CASES]
    ref = [host_bits(ops.q4_matmul(x, *w, ws=ws)) for x, w, ws in zip(xs, weights, wss)]
    torch.cuda.synchronize()

    errors = []

    def worker(tid):
        try:
            st = torch.cuda.Stream()
            # per thread its own outputs and workspaces (a workspace is not shared between concurrent calls)
            outs = [torch.empty((n, N), dtype=torch.float16, device="cuda") for K, N, n in CASES]
            my_ws = [ops.workspace(n, K, N) for K, N, n in CASES]
            order = list(range(len(CASES)))
            rng = np.random.default_rng(tid)
            for rep in range(6):
                rng.shuffle(order)
                with torch.cuda.stream(st):
                    for i in order:
                        ops.q4_matmul(xs[i], *weights[i], y=outs[i], ws=my_ws[i], stream=st)
                st.synchronize()
                for i in range(len(CASES)):
                    if not np.array_equal(host_bits(outs[i]), ref[i]):
                        errors.append((tid, rep, CASES[i]))
        except Exception as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
