"""GPU parity of relax_q4_matmul_fused (RMSNorm prologue, SiLU-mul and
residual epilogues) against the CPU oracle, on the decode GEMV (n <= 2) and
on the tensor-core path (n > 2, every token tile and split the planner picks
for these shapes), plus bitwise pins of the epilogues.

Reference: oracle.fused (plain numpy, fp16 at every tensor boundary of the
unfused program) around oracle.matmul_f64 (plain C, fp64).  Bar: the
north-star tolerance of tests/_util.py on the final output.
"""
import numpy as np
import pytest

import oracle
from oracle import fused as fo
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, assert_within_tol_f, dev_weights, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

R, S, Q = ops.OP_RMSNORM_X, ops.OP_SILU_MUL, ops.OP_RESIDUAL
EPS = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2311_02103_b200 import build
    build.build()
    ops.lib()


def reference(x_bits, packed, scales, K, N, op, gamma_bits, res_bits):
    xin = fo.rmsnorm_x(x_bits, gamma_bits, EPS) if op & R else x_bits
    r = oracle.matmul_f64(xin, packed, scales, K, N)
    v = fo.silu_mul(r) if op & S else r
    return fo.residual(v, res_bits) if op & Q else v


def run_fused(x_bits, packed, scales, op, gamma_bits, res_bits, inplace=False):
    n, K = x_bits.shape
    N = packed.shape[0]
    pw, sc = dev_weights(packed, scales)
    x = dev_x(x_bits)
    gamma = dev_x(gamma_bits[None, :])[0] if op & R else None
    n_out = N // 2 if op & S else N
    res = dev_x(res_bits) if op & Q else None
    nb = ops.plan_workspace_fused(n, K, N, op)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda") if nb else None
    if inplace:
        y = res
    else:
        y = torch.full((n, n_out), float("nan"), dtype=torch.float16, device="cuda")
    ops.q4_matmul_fused(x, pw, sc, y=y, rms_weight=gamma, rms_eps=EPS, silu_mul=bool(op & S),
                        residual=res, ws=ws)
    torch.cuda.synchronize()
    return host_bits(y)


def case(K, N, n, op, seed, kind="realistic"):
    packed, scales = inputs.weights(kind, seed, K, N)
    x = inputs.activations(seed + 1, n, K, "normal")
    rng = np.random.default_rng(seed + 2)
    gamma = rng.uniform(0.5, 1.5, K).astype(np.float16).view(np.uint16)
    n_out = N // 2 if op & S else N
    res = (rng.standard_normal((n, n_out)) * 0.05).astype(np.float16).view(np.uint16)
    return x, packed, scales, gamma, res


OPS = [R, S, Q, R | S, R | Q, S | Q, R | S | Q]
SHAPES = [(256, 256), (4096, 1024), (2048, 300), (11008, 512)]


@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("n", [1, 2, 3, 16, 64, 200])
def test_fused_parity(op, n):
    for i, (K, N) in enumerate(SHAPES):
        if n >= 64 and K * N > 4096 * 1024:
            continue
        x, packed, scales, gamma, res = case(K, N, n, op, 4000 + 10 * i + n)
        y = run_fused(x, packed, scales, op, gamma, res)
        want = reference(x, packed, scales, K, N, op, gamma, res)
        assert_within_tol(y, want, f"fused op={op} K={K} N={N} n={n} sched={ops.query_schedule(n, K, N)}")


@pytest.mark.parametrize("n", [1, 2, 5, 130])
def test_fused_llama_shapes_sampled(n):
    """7B shapes at full size: fused gate/up (N = 22016 interleaved) with SiLU-mul
    and RMSNorm, down-proj with the residual; compared on sampled columns."""
    for K, N, op in [(4096, 22016, R | S), (11008, 4096, Q), (4096, 12288, R)]:
        x, packed, scales, gamma, res = case(K, N, n, op, 4500 + n)
        y = run_fused(x, packed, scales, op, gamma, res).view(np.float16).astype(np.float64)
        rng = np.random.default_rng(n)
        n_out = N // 2 if op & S else N
        cols = np.sort(rng.choice(n_out, 64, replace=False))
        rows = np.stack([2 * cols, 2 * cols + 1], axis=1).reshape(-1) if op & S else cols
        xin = fo.rmsnorm_x(x, gamma, EPS) if op & R else x
        r = oracle.matmul_cols_f64(xin, packed, scales, K, rows)
        v = fo.silu_mul(r) if op & S else r
        want = fo.residual(v, res[:, cols]) if op & Q else v
        assert_within_tol_f(y[:, cols], want, f"fused 7B shape K={K} N={N} op={op} n={n}")


@pytest.mark.parametrize("n", [1, 2, 7, 100])
def test_residual_zero_weights_bitwise(n):
    """W = 0 (codes 7): y = fp16(+-0 + res) = res, bitwise, on every path."""
    K, N = 512, 384
    packed = np.full((N, K // 8), 0x77777777, dtype=np.uint32)
    scales = np.full((N, K // 32), 0x3C00, dtype=np.uint16)
    x = inputs.activations(9, n, K, "normal")
    res = (np.random.default_rng(1).standard_normal((n, N))).astype(np.float16).view(np.uint16)
    y = run_fused(x, packed, scales, Q, None, res)
    assert np.array_equal(y, res)
    y2 = run_fused(x, packed, scales, Q, None, res.copy(), inplace=True)     # residual == y
    assert np.array_equal(y2, res)


@pytest.mark.parametrize("n", [1, 2, 7, 100])
def test_silu_mul_zero_gate_bitwise(n):
    """gate rows W = 0 -> silu(0) * u = 0 for every pair, bitwise, on both the
    tensor path and the decode GEMV (whose factored zero point cancels an all-7
    group exactly)."""
    K, N = 512, 256
    packed, scales = inputs.weights("stress", 77, K, N)
    packed = packed.copy()
    packed[0::2] = 0x77777777                           # every gate row has codes 7
    x = inputs.activations(10, n, K, "normal")
    y = run_fused(x, packed, scales, S, None, None)
    assert np.all((y & 0x7FFF) == 0)


def test_fused_graph_chain():
    """A decoder-block-like chain of fused calls captured in a CUDA graph
    replays to the same bits as the eager chain."""
    K, N = 1024, 2048
    packed, scales = inputs.weights("realistic", 90, K, 2 * K)      # fused gate/up -> N/2 = K
    pd, sd = inputs.weights("realistic", 91, K, K)
    pw, sc = dev_weights(packed, scales)
    pw2, sc2 = dev_weights(pd, sd)
    x = dev_x(inputs.activations(11, 1, K, "normal"))
    gamma = torch.ones(K, dtype=torch.float16, device="cuda")
    h = torch.empty((1, K), dtype=torch.float16, device="cuda")
    out = torch.empty((1, K), dtype=torch.float16, device="cuda")
    st = torch.cuda.Stream()

    def chain():
        ops.q4_matmul_fused(x, pw, sc, y=h, rms_weight=gamma, silu_mul=True, stream=st)
        ops.q4_matmul_fused(h, pw2, sc2, y=out, residual=x, stream=st)

    with torch.cuda.stream(st):
        chain()
    torch.cuda.synchronize()
    eager = host_bits(out).copy()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        chain()
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(host_bits(out), eager)


def test_fused_workspace_shared_with_split_workspace_calls():
    """the tensor path's RMSNORM_X prologue writes the normalised x
    past the split-K ticket region, so one workspace can serve a fused call
    and then forced workspace split-K calls (which need zero tickets)."""
    K, N, n = 4096, 1024, 64
    x, packed, scales, gamma, _ = case(K, N, n, R, 7700)
    pw, sc = dev_weights(packed, scales)
    nb = max(ops.plan_workspace_fused(n, K, N, R), 4096 + 8 * n * N * 4)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    xd = dev_x(x)
    gd = dev_x(gamma[None, :])[0]
    cols = np.arange(0, N, 29)
    for rep in range(3):
        y = ops.q4_matmul_fused(xd, pw, sc, rms_weight=gd, rms_eps=EPS, ws=ws)
        assert ops.query_schedule(n, K, N)["variant"] == "tc"
        want = oracle.matmul_cols_f64(fo.rmsnorm_x(x, gamma, EPS), packed, scales, K, cols)
        assert_within_tol(host_bits(y)[:, cols], want, f"fused rmsnorm rep={rep}")
        y2 = ops.q4_matmul_ex(xd, pw, sc, ws=ws, variant=ops.VARIANT_TC, split_k=8, bn=64,
                              flags=ops.FLAG_SPLIT_WORKSPACE)
        torch.cuda.synchronize()
        assert_within_tol(host_bits(y2)[:, cols], oracle.matmul_cols_f64(x, packed, scales, K, cols),
                          f"split-workspace after fused rep={rep}")
