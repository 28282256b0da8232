"""GPU parity of decode attention over a symbolic KV length and of the KV
append (reading 21) against oracle/attention.py.

Tolerance as for the matmul (tests/_util.py): rel_F <= 2e-3 and max_rel <= 1e-2
with the row-RMS floor, per (sequence, head) output row; zero-length
sequences give exact zeros; reruns are bitwise identical."""
import numpy as np
import pytest

from oracle import attention as oa
from paper_2311_02103_b200 import ops
from tests._util import assert_within_tol, host_bits

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def make(batch, hq, hkv, lmax, seed):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((batch, hq, 128)).astype(np.float16)
    k = rng.standard_normal((batch, hkv, lmax, 128)).astype(np.float16)
    v = rng.standard_normal((batch, hkv, lmax, 128)).astype(np.float16)
    return q.view(np.uint16), k.view(np.uint16), v.view(np.uint16)


def dev16(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.float16)).cuda()


@pytest.mark.parametrize("hq,hkv", [(32, 32), (64, 8), (8, 2), (16, 4)])
@pytest.mark.parametrize("lens", [[1], [256], [257], [4096], [0, 5, 255, 1000], [4095, 3, 512]])
def test_attention_matches_oracle(hq, hkv, lens):
    lmax = max(max(lens), 1)
    batch = len(lens)
    q, k, v = make(batch, hq, hkv, lmax, seed=hq + lmax + batch)
    want = oa.attention_decode(q, k, v, lens, n_kv_heads=hkv)
    lt = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = ops.attn_decode(dev16(q), dev16(k), dev16(v), lt)
    torch.cuda.synchronize()
    got = host_bits(out)
    for b, L in enumerate(lens):
        if L == 0:
            assert np.all(got[b] == 0)
            continue
        assert_within_tol(got[b].reshape(hq, 128), want[b], f"attention hq={hq} hkv={hkv} L={L}")
    again = host_bits(ops.attn_decode(dev16(q), dev16(k), dev16(v), lt))
    assert np.array_equal(got, again)


def test_kv_append_then_attend_in_graph():
    """Append the new token's k, v at position len - 1 and attend over len keys,
    captured in a CUDA graph (as bench.py --kv runs it), against the oracle."""
    batch, hq, hkv, lmax = 2, 16, 4, 600
    q, k, v = make(batch, hq, hkv, lmax, seed=5)
    rng = np.random.default_rng(6)
    kn = rng.standard_normal((batch, hkv, 128)).astype(np.float16).view(np.uint16)
    vn = rng.standard_normal((batch, hkv, 128)).astype(np.float16).view(np.uint16)
    lens = [600, 333]
    pos = [L - 1 for L in lens]
    kc, vc = oa.kv_append(k, v, kn, vn, pos)
    want = oa.attention_decode(q, kc, vc, lens, n_kv_heads=hkv)
    dk, dv = dev16(k), dev16(v)
    dq, dkn, dvn = dev16(q), dev16(kn), dev16(vn)
    lt = torch.tensor(lens, dtype=torch.int32, device="cuda")
    pt = torch.tensor(pos, dtype=torch.int32, device="cuda")
    out = torch.empty((batch, hq, 128), dtype=torch.float16, device="cuda")
    ws = torch.empty(ops.attn_decode_workspace(batch, hq, lmax), dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ops.kv_append(dkn, dvn, pt, dk, dv, stream=st)
        ops.attn_decode(dq, dk, dv, lt, out=out, ws=ws, stream=st)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(host_bits(dk), kc) and np.array_equal(host_bits(dv), vc)
    got = host_bits(out)
    for b in range(batch):
        assert_within_tol(got[b], want[b], f"append+attend b={b}")


@pytest.mark.parametrize("n", [1, 2])
def test_kv_append_fused_into_qkv_epilogue(n):
    """RELAX_OP_KV_APPEND: the fused q/k/v projection (RMSNorm prologue) stores
    its key / value rows at each token's cache position while writing y:
    y is bit-identical to the same call without the op, the cache rows at the
    positions equal y's key / value slices bit for bit, nothing else in the
    caches changes, and out-of-range positions store nothing."""
    from paper_2311_02103_b200 import inputs
    from tests._util import dev_weights, dev_x
    hq, hkv, K, lmax = 8, 2, 512, 300
    N = (hq + 2 * hkv) * 128
    pk, sc = inputs.realistic_weights(6100 + n, K, N)
    w = dev_weights(pk, sc)
    x = dev_x(inputs.activations(6200 + n, n, K))
    gamma = torch.from_numpy(np.random.default_rng(1).uniform(0.5, 1.5, K).astype(np.float16)).cuda()
    rng = np.random.default_rng(7)
    k0 = rng.standard_normal((n, hkv, lmax, 128)).astype(np.float16)
    v0 = rng.standard_normal((n, hkv, lmax, 128)).astype(np.float16)
    for pos in ([299, 17][:n], [0, -1][:n], [lmax, 5][:n]):
        kc, vc = torch.from_numpy(k0.copy()).cuda(), torch.from_numpy(v0.copy()).cuda()
        pt = torch.tensor(pos, dtype=torch.int32, device="cuda")
        y = ops.q4_matmul_fused(x, *w, rms_weight=gamma, kv_append=(kc, vc, pt, hq * 128))
        y_ref = ops.q4_matmul_fused(x, *w, rms_weight=gamma)
        torch.cuda.synchronize()
        yb = host_bits(y)
        assert np.array_equal(yb, host_bits(y_ref))
        kb, vb = host_bits(kc), host_bits(vc)
        kw, vw = k0.view(np.uint16).copy(), v0.view(np.uint16).copy()
        for t, p in enumerate(pos):
            if 0 <= p < lmax:
                kw[t, :, p, :] = yb[t, hq * 128:(hq + hkv) * 128].reshape(hkv, 128)
                vw[t, :, p, :] = yb[t, (hq + hkv) * 128:].reshape(hkv, 128)
        assert np.array_equal(kb, kw) and np.array_equal(vb, vw), pos
