"""GPU parity over every automatic schedule class (verdict r1 "parity coverage").

For each weight shape of configs c1-c5, the rank shards of the 2/4/8-way
Megatron split of the 70B set, and the fused q/k/v, gate/up layouts, the
dispatch (relax_query_schedule, P:409-413 -- n symbolic, K and N static) is
enumerated over n in [1, 4096]; every distinct (variant, tile, split-K) class
is run at the first and the last n that selects it, through the public
relax_q4_matmul_ws, and compared with the fp64 oracle: all rows for n <= 64,
16 sampled rows (always the first and the last) otherwise, on sampled output
columns (always the first and the last, i.e. the ragged tail).  Tolerance:
BASELINE.json north_star (rel_F <= 2e-3, max_rel <= 1e-2), tests/_util.py.
"""
import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

N_MAX = 4096


def _llama_shapes():
    out = []
    for model in ("llama2-7b", "llama2-13b", "llama2-70b"):
        spec = inputs.LLAMA_SETS[model]
        d = {nm: (K, N) for nm, K, N in spec["mats"]}
        for nm, K, N in spec["mats"]:
            out.append((f"{model}.{nm}", K, N))
        out.append((f"{model}.lm_head", *spec["lm_head"]))
        K = d["q"][0]
        out.append((f"{model}.qkv_fused", K, d["q"][1] + d["k"][1] + d["v"][1]))
        out.append((f"{model}.gate_up_fused", K, d["gate"][1] + d["up"][1]))
    spec = inputs.LLAMA_SETS["llama2-70b"]
    for p in (2, 4, 8):
        for nm, K, N in spec["mats"] + [("lm_head", *spec["lm_head"])]:
            if nm in ("o", "down"):
                out.append((f"70b.tp{p}.{nm}", K // p, N))
            else:
                out.append((f"70b.tp{p}.{nm}", K, N // p))
    out.append(("c1", 256, 256))
    seen, uniq = set(), []
    for name, K, N in out:
        if (K, N) not in seen:
            seen.add((K, N))
            uniq.append((name, K, N))
    return uniq


SHAPES = _llama_shapes()


def schedule_classes(K, N, n_max=N_MAX):
    """{class: [first n, last n]} of the automatic schedule over n in [1, n_max]."""
    cls = {}
    for n in range(1, n_max + 1):
        s = ops.query_schedule(n, K, N)
        key = (s["variant"], s["tile"], s["split_k"], s.get("persistent", False), s.get("stream_k", False),
               s.get("two_part", False), s.get("two_part_persistent", False))
        if key not in cls:
            cls[key] = [n, n]
        cls[key][1] = n
    return cls


def check_ns(name, K, N, ns, seed, kind="stress"):
    packed, scales = inputs.weights(kind, seed, K, N)
    pw, sc = dev_weights(packed, scales)
    nmax = max(ns)
    xall = inputs.activations(seed + 1, nmax, K, "uniform" if kind == "stress" else "normal")
    xd = dev_x(xall)
    ws = ops.workspace(nmax, K, N)
    rng = np.random.default_rng(seed)
    cols = np.unique(np.concatenate([[0, N - 1], rng.choice(N, size=min(N, 46), replace=False)]))
    for n in sorted(set(ns)):
        y = host_bits(ops.q4_matmul(xd[:n], pw, sc, ws=ws))
        rows = np.arange(n) if n <= 64 else np.unique(np.concatenate([[0, n - 1], rng.choice(n, 14, replace=False)]))
        r = oracle.matmul_cols_f64(xall[rows], packed, scales, K, cols)
        assert_within_tol(y[rows][:, cols], r, f"{name} {K}x{N} n={n} sched={ops.query_schedule(n, K, N)}")


@pytest.mark.parametrize("name,K,N", SHAPES, ids=[f"{nm}-{K}x{N}" for nm, K, N in SHAPES])
def test_every_schedule_class(name, K, N):
    cls = schedule_classes(K, N)
    ns = sorted({n for lo_hi in cls.values() for n in lo_hi})
    check_ns(name, K, N, ns, seed=9000 + (K * 7 + N) % 997)


@pytest.mark.parametrize("K,N", [(96, 200), (4128, 1000), (2080, 72)])
def test_k_not_multiple_of_256_auto(K, N):
    """K % 256 != 0 goes through the automatic dispatch to the generic
    CUDA-core GEMV at any n (the tensor path needs K % 256 == 0)."""
    check_ns("k-ragged", K, N, [1, 2, 3, 17, 300], seed=9500 + K, kind="realistic")
    for n in (1, 3, 17, 300):
        assert ops.query_schedule(n, K, N)["variant"] == "gemv"


def test_wide_lm_head_decode():
    """A 405B-class lm_head (K = 16384, N = 128256): the decode schedule fits
    the device (no RELAX_ERR_CUDA on legal shapes)."""
    check_ns("wide-lm-head", 16384, 128256, [1, 2], seed=9700)


def test_two_threads_two_streams():
    """Two host threads drive the library concurrently on their own streams
    (reentrant boundary, include/relax_q4.h); every result equals the serial
    one bitwise."""
    import threading
    K, N = 4096, 4096
    packed, scales = inputs.realistic_weights(9800, K, N)
    pw, sc = dev_weights(packed, scales)
    cases = [dev_x(inputs.activations(9801 + n, n, K)) for n in (1, 2, 5, 16, 64, 300)]
    serial = [host_bits(ops.q4_matmul(x, pw, sc, ws=ops.workspace(x.shape[0], K, N))) for x in cases]
    errors = []

    def worker(tid):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for rep in range(20):
                    for x, want in zip(cases, serial):
                        ws = ops.workspace(x.shape[0], K, N)
                        y = ops.q4_matmul(x, pw, sc, ws=ws, stream=st)
                        st.synchronize()
                        if not np.array_equal(host_bits(y), want):
                            errors.append((tid, rep, x.shape[0]))
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:5]
