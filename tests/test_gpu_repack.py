"""GPU parity of relax_q4_repack: the device conversion of a
KN-layout or G = 64 / 128 weight into the native format equals the oracle's
plain definition (oracle/formats.py) bit for bit, and the converted weight
feeds the matmul, checked against the fp64 oracle."""
import numpy as np
import pytest

import oracle
from oracle import formats as fm
from paper_2311_02103_b200 import inputs, ops
from tests._util import assert_within_tol, dev_x, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def src_format(K, N, layout, group, seed):
    rng = np.random.default_rng(seed)
    q = rng.integers(0, 16, size=(N, K), dtype=np.uint8)
    sg = rng.uniform(2.0 ** -10, 2.0 ** -5, size=(N, K // group)).astype(np.float16).view(np.uint16)
    p = inputs.pack_codes(q)                              # native-order words [N][K/8]
    if layout == "nk":
        return p, sg
    return np.ascontiguousarray(p.T), np.ascontiguousarray(sg.T)


@pytest.mark.parametrize("layout", ["nk", "kn"])
@pytest.mark.parametrize("group", [32, 64, 128])
@pytest.mark.parametrize("K,N", [(256, 24), (4096, 1000), (11008, 512)])
def test_repack_bit_exact_and_matmul(layout, group, K, N):
    src_p, src_s = src_format(K, N, layout, group, seed=K + N + group)
    want_p, want_s = fm.to_native(src_p, src_s, K, N, layout, group)
    dp = torch.from_numpy(src_p.view(np.int32)).cuda()
    ds = torch.from_numpy(src_s.view(np.float16)).cuda()
    pw, sc = ops.q4_repack(dp, ds, K, N, layout=layout, group=group)
    torch.cuda.synchronize()
    assert np.array_equal(pw.cpu().numpy().view(np.uint32), want_p)
    assert np.array_equal(host_bits(sc), want_s)
    # the converted weight in the matmul (decode and a tensor-core n)
    for n in (1, 64):
        x = inputs.activations(n + K, n, K)
        y = host_bits(ops.q4_matmul(dev_x(x), pw, sc, ws=ops.workspace(n, K, N)))
        cols = np.arange(0, N, max(1, N // 40))
        r = oracle.matmul_cols_f64(x, want_p, want_s, K, cols)
        assert_within_tol(y[:, cols], r, f"repacked {layout} G={group} {K}x{N} n={n}")


@pytest.mark.parametrize("group", [32, 128])
@pytest.mark.parametrize("K,N", [(256, 24), (4096, 1000), (11008, 300)])
def test_repack_q3_bit_exact_and_matmul(group, K, N):
    """3-bit source (layout "nk3", reading 20): random words (every 96-bit
    pattern is a valid code triple) -> native words equal the oracle's
    to_native bit for bit, and the matmul on them matches the oracle of the
    3-bit weight."""
    rng = np.random.default_rng(K + N + group)
    src_p = rng.integers(0, 2 ** 32, size=(N, K // 32 * 3), dtype=np.uint64).astype(np.uint32)
    src_s = rng.uniform(2.0 ** -10, 2.0 ** -5, size=(N, K // group)).astype(np.float16).view(np.uint16)
    want_p, want_s = fm.to_native(src_p, src_s, K, N, "nk3", group)
    pw, sc = ops.q4_repack(torch.from_numpy(src_p.view(np.int32)).cuda(), torch.from_numpy(src_s.view(np.float16)).cuda(),
                           K, N, layout="nk3", group=group)
    torch.cuda.synchronize()
    assert np.array_equal(pw.cpu().numpy().view(np.uint32), want_p)
    assert np.array_equal(host_bits(sc), want_s)
    W3 = fm.dequant3(src_p, src_s, K, N, group).view(np.float16).astype(np.float64)   # [N][K]
    for n in (1, 64):
        x = inputs.activations(n + K + 3, n, K)
        y = host_bits(ops.q4_matmul(dev_x(x), pw, sc, ws=ops.workspace(n, K, N)))
        r = x.view(np.float16).astype(np.float64) @ W3.T
        assert_within_tol(y, r, f"repacked nk3 G={group} {K}x{N} n={n}")
