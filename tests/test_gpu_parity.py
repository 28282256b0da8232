"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): dequantised weights bit-exact; outputs
within rel_F <= 2e-3 and max_rel <= 1e-2 of the oracle's fp64 sum.  Pinned
invariants (one-hot extraction, identity scale, zeros) are bitwise.
"""
import numpy as np
import pytest

import oracle
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2311_02103_b200 import build
    build.build()
    ops.lib()


def run(x_bits, packed, scales, variant=0, split_k=0, bn=0, ws_n_max=None, flags=0):
    x = dev_x(x_bits)
    pw, sc = dev_weights(packed, scales)
    n, K = x.shape
    N = pw.shape[0]
    ws = None
    if (split_k > 1 and flags & ops.FLAG_SPLIT_WORKSPACE) or ws_n_max:
        nb = max(ops.plan_workspace(ws_n_max or n, K, N), split_k * n * N * 4 + 4096)
        ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    y = torch.full((n, N), float("nan"), dtype=torch.float16, device="cuda")
    ops.q4_matmul_ex(x, pw, sc, y=y, ws=ws, variant=variant, split_k=split_k, bn=bn, flags=flags)
    torch.cuda.synchronize()
    return host_bits(y)


# ------------------------------------------------------------------ dequant
def test_dequant_exhaustive_bit_exact():
    """16 codes x 65536 scale bit patterns, GPU export == oracle, bitwise."""
    N, K = 65536, 32
    codes = np.tile(np.concatenate([np.arange(16), np.arange(16)]), (N, 1)).astype(np.uint8)
    packed = inputs.pack_codes(codes)
    scales = np.arange(N, dtype=np.uint32).astype(np.uint16).reshape(N, 1)
    want = oracle.dequant(packed, scales, K, N)
    pw, sc = dev_weights(packed, scales)
    got = host_bits(ops.q4_dequant(pw, sc, K))
    nan_w = np.isnan(want.view(np.float16))
    nan_g = np.isnan(got.view(np.float16))
    assert np.array_equal(nan_w, nan_g)
    assert np.array_equal(got[~nan_g], want[~nan_w])


@pytest.mark.parametrize("kind", ["realistic", "stress"])
def test_dequant_llama_shape_bit_exact(kind):
    K, N = 4096, 1024
    packed, scales = inputs.weights(kind, 1002, K, N)
    want = oracle.dequant(packed, scales, K, N)
    pw, sc = dev_weights(packed, scales)
    got = host_bits(ops.q4_dequant(pw, sc, K))
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("kind", ["realistic", "stress"])
@pytest.mark.parametrize("n", [1, 4])
def test_config1_auto(kind, n):
    K = N = 256
    packed, scales = inputs.weights(kind, 1000, K, N)
    x = inputs.activations(7 + n, n, K, "normal" if kind == "realistic" else "uniform")
    r = oracle.matmul_f64(x, packed, scales, K, N)
    y = run(x, packed, scales)
    assert_within_tol(y, r, f"c1 {kind} n={n}")


WSF = 2   # RELAX_FLAG_SPLIT_WORKSPACE
VARIANTS = [("gemv", 1, 0, 0, 0), ("smalln", 3, 0, 0, 0), ("tc16", 2, 1, 16, 0), ("tc32", 2, 1, 32, 0), ("tc64", 2, 1, 64, 0),
            ("tc128", 2, 1, 128, 0), ("tc256", 2, 1, 256, 4), ("tc256p", 2, 1, 256, 0),
            ("tc16s3c", 2, 3, 16, 0), ("tc64s2c", 2, 2, 64, 0), ("tc128s2c", 2, 2, 128, 0),
            ("tc256s3c", 2, 3, 256, 0),
            ("tc16s3w", 2, 3, 16, WSF), ("tc64s2w", 2, 2, 64, WSF), ("tc128s2w", 2, 2, 128, WSF)]


@pytest.mark.parametrize("name,variant,split,bn,flags", VARIANTS)
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 9, 16, 17, 33, 64, 100, 129, 257, 300])
def test_every_variant_ragged(name, variant, split, bn, flags, n):
    """Several M tiles and a ragged tail (N = 328 = 2*128 + 72), 3 weight
    stages of 256 k (K = 768), ragged token tiles."""
    if name in ("gemv", "smalln") and n > 17:
        pytest.skip("GEMV / small-n kernels exercised at small n")
    K, N = 768, 328
    packed, scales = inputs.realistic_weights(2000, K, N)
    x = inputs.activations(7 + n, n, K)
    r = oracle.matmul_f64(x, packed, scales, K, N)
    y = run(x, packed, scales, variant=variant, split_k=split, bn=bn, flags=flags)
    assert_within_tol(y, r, f"{name} n={n}")


@pytest.mark.parametrize("name,variant,split,bn,flags", VARIANTS)
def test_one_hot_extraction_bitwise(name, variant, split, bn, flags):
    """x row i = e_{k_i} -> y[i,:] == W[k_i,:] bitwise (exact product, exact
    zero sums, one rounding of an fp16 value)."""
    K, N = 512, 256
    packed, scales = inputs.stress_weights(2100, K, N)
    ks = [0, 1, 7, 8, 31, 32, 255, 256, 300, 511, 63, 64, 127, 128, 200, 400, 5]
    x = np.zeros((len(ks), K), dtype=np.uint16)
    for i, k in enumerate(ks):
        x[i, k] = 0x3C00
    W = oracle.dequant(packed, scales, K, N)          # [N][K]
    y = run(x, packed, scales, variant=variant, split_k=split, bn=bn, flags=flags)
    for i, k in enumerate(ks):
        assert np.array_equal(y[i], W[:, k]), f"{name}: row for k={k}"


@pytest.mark.parametrize("name,variant,split,bn,flags", VARIANTS)
def test_identity_scale_integer_exact(name, variant, split, bn, flags):
    """scales = 1, x in {-1,0,1}: every partial sum is an integer < 2^24, so y
    is exact in any summation order."""
    K, N, n = 1024, 200, 12
    g = np.random.default_rng(77)
    packed = g.integers(0, 2**32, size=(N, K // 8), dtype=np.uint64).astype(np.uint32)
    scales = np.full((N, K // 32), 0x3C00, dtype=np.uint16)
    xi = g.integers(-1, 2, size=(n, K))
    x = xi.astype(np.float16).view(np.uint16)
    r = oracle.matmul_f64(x, packed, scales, K, N)
    assert np.all(np.abs(r) <= 2048)
    y = run(x, packed, scales, variant=variant, split_k=split, bn=bn, flags=flags)
    assert np.array_equal(y.view(np.float16).astype(np.float64), r)


@pytest.mark.parametrize("case", ["codes7", "scales0", "x0"])
@pytest.mark.parametrize("name,variant,split,bn,flags", VARIANTS)
def test_zero_invariants(case, name, variant, split, bn, flags):
    K, N, n = 512, 256, 5
    packed, scales = inputs.stress_weights(2200, K, N)
    x = inputs.activations(2201, n, K)
    if case == "codes7":
        packed = np.full_like(packed, 0x77777777)
    elif case == "scales0":
        scales = np.zeros_like(scales)
    else:
        x = np.zeros_like(x)
    y = run(x, packed, scales, variant=variant, split_k=split, bn=bn, flags=flags)
    # r == 0 => y == +-0 bitwise for every variant (reading 10)
    assert np.all((y & 0x7FFF) == 0)


def test_n_zero_is_noop():
    K, N = 256, 256
    packed, scales = inputs.stress_weights(1, K, N)
    pw, sc = dev_weights(packed, scales)
    x = torch.empty((0, K), dtype=torch.float16, device="cuda")
    y = torch.empty((0, N), dtype=torch.float16, device="cuda")
    ops.q4_matmul(x, pw, sc, y=y)
    torch.cuda.synchronize()


def test_deterministic_reruns_bitwise():
    K, N = 4096, 4096
    packed, scales = inputs.realistic_weights(1001, K, N)
    pw, sc = dev_weights(packed, scales)
    for n in (1, 3, 16, 40, 200, 1000):
        x = dev_x(inputs.activations(7 + n, n, K))
        ws = ops.workspace(n, K, N)
        a = host_bits(ops.q4_matmul(x, pw, sc, ws=ws))
        b = host_bits(ops.q4_matmul(x, pw, sc, ws=ws))
        assert np.array_equal(a, b), f"n={n}"


# ------------------------------------------------------------------ full sizes
def test_prefix_sweep_4096_sampled_columns():
    """One n=4096 input pins every n in [1, 4096] (rows are independent):
    each call with x[:n] is compared with the oracle's rows r[:n] on 48
    sampled output columns, in the auto-dispatch launch configuration."""
    K, N = 4096, 4096
    packed, scales = inputs.realistic_weights(3001, K, N)
    xall = inputs.activations(7 + 4096, 4096, K)
    g = np.random.default_rng(0)
    cols = np.sort(g.choice(N, size=48, replace=False))
    r = oracle.matmul_cols_f64(xall, packed, scales, K, cols)
    pw, sc = dev_weights(packed, scales)
    xd = dev_x(xall)
    ws = ops.workspace(4096, K, N)
    ns = list(range(1, 17)) + [24, 32, 48, 64, 80, 96, 100, 128, 192, 256, 384, 512, 768,
                                1000, 1024, 1536, 2048, 3072, 4095, 4096, 17]
    for n in ns:
        y = host_bits(ops.q4_matmul(xd[:n], pw, sc, ws=ws))
        assert_within_tol(y[:, cols], r[:n], f"prefix n={n}")


@pytest.mark.parametrize("K,N", [(4096, 11008), (11008, 4096), (4096, 32000), (5120, 13824),
                                 (13824, 5120), (8192, 1024), (28672, 8192)])
@pytest.mark.parametrize("n", [1, 16, 512])
def test_llama_shapes_sampled(K, N, n):
    packed, scales = inputs.realistic_weights(4000 + K % 97 + N % 89, K, N)
    x = inputs.activations(7 + n, n, K)
    g = np.random.default_rng(1)
    cols = np.sort(g.choice(N, size=32, replace=False))
    rows = np.arange(n) if n <= 16 else np.sort(g.choice(n, size=16, replace=False))
    r = oracle.matmul_cols_f64(x[rows], packed, scales, K, cols)
    pw, sc = dev_weights(packed, scales)
    ws = ops.workspace(n, K, N)
    y = host_bits(ops.q4_matmul(dev_x(x), pw, sc, ws=ws))
    assert_within_tol(y[rows][:, cols], r, f"{K}x{N} n={n}")


def test_cuda_graph_capture_every_variant():
    """Calls are capturable (no allocation, no host sync inside) and the
    replayed graph reproduces the eager result bitwise."""
    K, N = 4096, 4096
    packed, scales = inputs.realistic_weights(5001, K, N)
    pw, sc = dev_weights(packed, scales)
    ns = [1, 2, 16, 64, 300]
    xs = [dev_x(inputs.activations(7 + n, n, K)) for n in ns]
    ws = ops.workspace(max(ns), K, N)
    eager = [host_bits(ops.q4_matmul(x, pw, sc, ws=ws)) for x in xs]
    ys = [torch.empty((n, N), dtype=torch.float16, device="cuda") for n in ns]
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for x, y in zip(xs, ys):
            ops.q4_matmul(x, pw, sc, y=y, ws=ws)
    g.replay()
    torch.cuda.synchronize()
    for e, y in zip(eager, ys):
        assert np.array_equal(e, host_bits(y))


def test_workspace_reused_across_calls():
    """One zero-filled workspace serves a sequence of forced workspace split-K
    calls of different n (the tickets reset themselves), each within tolerance."""
    K, N = 8192, 1024
    pw_np, sc_np = inputs.realistic_weights(6001, K, N)
    pw, sc = dev_weights(pw_np, sc_np)
    ws = torch.zeros(4096 + 12 * 64 * N * 4, dtype=torch.uint8, device="cuda")
    cols = np.arange(0, N, 37)
    for n, split in ((16, 12), (17, 9), (40, 12), (64, 10), (16, 12), (33, 11), (5, 12)):
        xb = inputs.activations(n, n, K)
        y = host_bits(ops.q4_matmul_ex(dev_x(xb), pw, sc, ws=ws, variant=ops.VARIANT_TC,
                                       split_k=split, flags=ops.FLAG_SPLIT_WORKSPACE))
        r = oracle.matmul_cols_f64(xb, pw_np, sc_np, K, cols)
        assert_within_tol(y[:, cols], r, f"reuse n={n} split={split}")


@pytest.mark.parametrize("n", [1, 2, 3, 64, 300])
def test_dependent_pdl_chain_in_graph(n):
    """The benchmark's launch configuration with a REAL data dependency: a
    chain y1 = W1 x, y2 = W2 y1, y3 = W3 y2 (square shapes, K = N) launched
    back to back with programmatic dependent launch inside one CUDA graph,
    replayed several times.  Each kernel prefetches its weights before
    griddepcontrol.wait; this checks that x is only read after the previous
    kernel's y is complete: every stage matches the oracle applied to the
    previous stage's GPU output (fp16, as the chain passes it)."""
    K = 1024
    mats = [inputs.weights("realistic", 7100 + i, K, K) for i in range(3)]
    dev = [dev_weights(p, s) for p, s in mats]
    x0 = inputs.activations(7200 + n, n, K)
    x = dev_x(x0)
    ys = [torch.empty((n, K), dtype=torch.float16, device="cuda") for _ in range(3)]
    ws = ops.workspace(n, K, K)
    st = torch.cuda.Stream()

    def chain():
        inp = x
        for (pw, sc), y in zip(dev, ys):
            ops.q4_matmul(inp, pw, sc, y=y, ws=ws, stream=st)
            inp = y

    with torch.cuda.stream(st):
        chain()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        chain()
    for y in ys:
        y.fill_(float("nan"))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    inp_bits = x0
    for i, ((packed, scales), y) in enumerate(zip(mats, ys)):
        got = host_bits(y)
        r = oracle.matmul_f64(inp_bits, packed, scales, K, K)
        assert_within_tol(got, r, f"chain stage {i} n={n}")
        inp_bits = got


def test_random_shapes_every_path():
    """Seeded random (n, K, N) over the whole dispatch range, including tiny
    and ragged N (N < 8, N % 8 != 0: no TMA store), K at the tensor-core
    minimum, and n just past tile sizes; the automatic schedule against the
    oracle."""
    rng = np.random.default_rng(20261018)
    cases = []
    for _ in range(24):
        K = int(rng.choice([256, 512, 768, 1280, 2304, 4096]))
        N = int(rng.choice([1, 2, 6, 8, 24, 130, 256, 384, 1000, 2048]))
        n = int(rng.choice([1, 2, 3, 7, 16, 17, 33, 64, 65, 129, 200, 257]))
        cases.append((n, K, N))
    cases += [(300, 256, 8), (1, 256, 1), (2, 4096, 6), (129, 1280, 130)]
    for i, (n, K, N) in enumerate(cases):
        packed, scales = inputs.weights("realistic" if i % 2 else "stress", 8000 + i, K, N)
        x = inputs.activations(8100 + i, n, K, "normal" if i % 2 else "uniform")
        r = oracle.matmul_f64(x, packed, scales, K, N)
        y = run(x, packed, scales, ws_n_max=n)
        assert_within_tol(y, r, f"random case {i}: n={n} K={K} N={N} sched={ops.query_schedule(n, K, N)}")


@pytest.mark.parametrize("layout", ["plain", "fused"])
@pytest.mark.parametrize("n", [1, 8, 32])
def test_bench_configuration_sampled(layout, n):
    """bench.py's launch configuration at full size: one decoder layer of the
    7B set (q, k, v, o, gate, up, down -- or, in the fused layout bench.py
    --fused times, qkv 4096x12288, o, gate_up 4096x22016, down) + lm_head,
    distinct weight buffers, n tokens (1 = decode, 8/32 = the batched-decode
    lines: small-n tensor path with cluster split-K), back-to-back calls with
    PDL captured in a CUDA graph and replayed; every output checked on sampled
    columns (all n rows) against the oracle."""
    spec = inputs.LLAMA_SETS["llama2-7b"]
    if layout == "fused":
        d = {name: (K, N) for name, K, N in spec["mats"]}
        mats = [("qkv", 4096, d["q"][1] + d["k"][1] + d["v"][1]), ("o", *d["o"]),
                ("gate_up", 4096, d["gate"][1] + d["up"][1]), ("down", *d["down"])]
    else:
        mats = list(spec["mats"])
    mats.append(("lm_head", *spec["lm_head"]))
    st = torch.cuda.Stream()
    host, devw, xs, ys = [], [], {}, []
    for i, (name, K, N) in enumerate(mats):
        pk, sc = inputs.realistic_weights(2000 + i, K, N)
        host.append((pk, sc))
        devw.append(dev_weights(pk, sc))
        if K not in xs:
            xs[K] = inputs.activations(2100 + K + n, n, K)
        ys.append(torch.full((n, N), float("nan"), dtype=torch.float16, device="cuda"))
    xd = {K: dev_x(v) for K, v in xs.items()}

    def step():
        for (name, K, N), (pw, sc), y in zip(mats, devw, ys):
            ops.q4_matmul_ex(xd[K], pw, sc, y=y, stream=st)

    with torch.cuda.stream(st):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        step()
    for y in ys:
        y.fill_(float("nan"))
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    for (name, K, N), (pk, sc), y in zip(mats, host, ys):
        cols = np.sort(rng.choice(N, 96, replace=False))
        r = oracle.matmul_cols_f64(xs[K], pk, sc, K, cols)
        assert_within_tol(host_bits(y)[:, cols], r,
                          f"bench config {layout} n={n} {name} {K}x{N} sched={ops.query_schedule(n, K, N)}")
