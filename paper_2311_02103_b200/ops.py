"""Python binding of the C-ABI in include/relax_q4.h (argument marshalling only).

Every function here forwards torch tensors' device pointers, sizes and the
current CUDA stream to librelax_q4.so; every step of the computation runs in
the library's sm_100a kernels.  There is no fallback: if the shared library
is missing or a call fails, a RelaxError is raised.

Names follow the ABI: relax_q4_matmul -> q4_matmul, relax_plan_workspace ->
plan_workspace, relax_q4_dequant -> q4_dequant, relax_query_schedule ->
query_schedule, relax_q4_matmul_ex -> q4_matmul_ex.

Tensor conventions:
    x         torch.float16 [n, K]          (contiguous, CUDA)
    packed_w  torch.int32   [N, K // 8]     (uint32 bit patterns stored as int32)
    scales    torch.float16 [N, K // 32]
    y         torch.float16 [n, N]
"""
from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# RELAX_Q4_LIB points the binding at another build of the same ABI (the
# experiments library of `build --experiments`, used by tools/ only).
LIB_PATH = os.environ.get("RELAX_Q4_LIB") or os.path.join(PKG, "librelax_q4.so")

RELAX_OK = 0
STATUS = {
    0: "RELAX_OK", 1: "RELAX_ERR_INVALID_ARG", 2: "RELAX_ERR_UNSUPPORTED_SHAPE",
    3: "RELAX_ERR_MISALIGNED", 4: "RELAX_ERR_ALIAS", 5: "RELAX_ERR_WORKSPACE",
    6: "RELAX_ERR_DEVICE", 7: "RELAX_ERR_CUDA",
}
VARIANT_AUTO, VARIANT_GEMV, VARIANT_TC, VARIANT_SMALLN = 0, 1, 2, 3
FLAG_NO_PDL = 1
FLAG_SPLIT_WORKSPACE = 2
FLAG_TILE_PER_CTA = 4

# every symbol include/relax_q4.h declares
EXPORTS = ("relax_plan_workspace", "relax_q4_matmul", "relax_q4_matmul_ws", "relax_q4_matmul_ex",
           "relax_query_schedule", "relax_q4_dequant", "relax_status_str", "relax_version",
           "relax_plan_workspace_fused", "relax_q4_matmul_fused", "relax_q4_repack",
           "relax_attn_decode_workspace", "relax_attn_decode", "relax_kv_append", "relax_q4_matmul_grouped",
           "relax_tp_comm_bytes", "relax_q4_matmul_allreduce")
# the persistent decode chain: experiments build only (include/relax_q4_debug.h)
CHAIN_EXPORTS = ("relax_q4_chain_workspace", "relax_q4_chain_init", "relax_q4_chain_run")

# fused neighbours (include/relax_q4.h RELAX_OP_*)
OP_RMSNORM_X, OP_SILU_MUL, OP_RESIDUAL, OP_KV_APPEND = 1, 2, 4, 8


class Fusion(ctypes.Structure):
    """struct relax_q4_fusion."""
    _fields_ = [("ops", ctypes.c_uint32), ("rms_eps", ctypes.c_float),
                ("rms_weight", ctypes.c_void_p), ("residual", ctypes.c_void_p),
                ("k_cache", ctypes.c_void_p), ("v_cache", ctypes.c_void_p), ("kv_pos", ctypes.c_void_p),
                ("kv_len_max", ctypes.c_int64), ("kv_heads", ctypes.c_int32), ("kv_row0", ctypes.c_int32)]


TP_MAX_WORLD = 8


class TpComm(ctypes.Structure):
    """struct relax_tp_comm: bufs[p] = rank p's exchange buffer mapped on this device."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("bufs", ctypes.c_void_p * TP_MAX_WORLD), ("buf_bytes", ctypes.c_size_t)]


class ChainOp(ctypes.Structure):
    """struct relax_q4_chain_op."""
    _fields_ = [("x", ctypes.c_void_p), ("packed_w", ctypes.c_void_p), ("scales", ctypes.c_void_p),
                ("y", ctypes.c_void_p), ("K", ctypes.c_int64), ("N", ctypes.c_int64), ("after", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class RelaxError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib().relax_status_str(status).decode()
        super().__init__(f"{where}: {msg}")


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load librelax_q4.so (built by paper_2311_02103_b200.build).  Raises if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not built: run `python -m paper_2311_02103_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, SZ, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
        L.relax_plan_workspace.argtypes = [I64, I64, I64, ctypes.POINTER(SZ)]
        L.relax_plan_workspace.restype = I
        L.relax_q4_matmul.argtypes = [P, I64, I64, I64, P, P, P, P]
        L.relax_q4_matmul.restype = I
        L.relax_q4_matmul_ws.argtypes = [P, I64, I64, I64, P, P, P, P, SZ, P]
        L.relax_q4_matmul_ws.restype = I
        L.relax_q4_matmul_ex.argtypes = [P, I64, I64, I64, P, P, P, P, SZ, I, I, I, ctypes.c_uint, P]
        L.relax_q4_matmul_ex.restype = I
        L.relax_query_schedule.argtypes = [I64, I64, I64, ctypes.POINTER(I), ctypes.POINTER(I),
                                           ctypes.POINTER(I), ctypes.POINTER(SZ), ctypes.POINTER(I)]
        L.relax_query_schedule.restype = I
        L.relax_q4_dequant.argtypes = [P, P, I64, I64, P, P]
        L.relax_q4_dequant.restype = I
        L.relax_status_str.argtypes = [I]
        L.relax_status_str.restype = ctypes.c_char_p
        L.relax_version.argtypes = []
        L.relax_version.restype = ctypes.c_char_p
        L.relax_plan_workspace_fused.argtypes = [I64, I64, I64, ctypes.c_uint32, ctypes.POINTER(SZ)]
        L.relax_plan_workspace_fused.restype = I
        L.relax_q4_matmul_fused.argtypes = [P, I64, I64, I64, P, P, P, ctypes.POINTER(Fusion), P, SZ, P]
        L.relax_q4_matmul_fused.restype = I
        L.relax_q4_repack.argtypes = [P, P, I64, I64, I, I, P, P, P]
        L.relax_q4_repack.restype = I
        L.relax_q4_matmul_grouped.argtypes = [P, I64, I64, I, ctypes.POINTER(I64), ctypes.POINTER(P),
                                              ctypes.POINTER(P), ctypes.POINTER(P), P]
        L.relax_q4_matmul_grouped.restype = I
        L.relax_attn_decode_workspace.argtypes = [I64, I64, I64, ctypes.POINTER(SZ)]
        L.relax_attn_decode_workspace.restype = I
        L.relax_attn_decode.argtypes = [P, P, P, P, I64, I64, I64, I64, I64, P, P, SZ, P]
        L.relax_attn_decode.restype = I
        L.relax_kv_append.argtypes = [P, P, P, I64, I64, I64, I64, P, P, P]
        L.relax_kv_append.restype = I
        if hasattr(L, "relax_q4_chain_run"):
            L.relax_q4_chain_workspace.argtypes = [I, ctypes.POINTER(SZ)]
            L.relax_q4_chain_workspace.restype = I
            L.relax_q4_chain_init.argtypes = [ctypes.POINTER(ChainOp), I, P, SZ]
            L.relax_q4_chain_init.restype = I
            L.relax_q4_chain_run.argtypes = [P, P]
            L.relax_q4_chain_run.restype = I
        L.relax_tp_comm_bytes.argtypes = [ctypes.c_int32, I64, ctypes.POINTER(SZ)]
        L.relax_tp_comm_bytes.restype = I
        L.relax_q4_matmul_allreduce.argtypes = [ctypes.POINTER(TpComm), P, I64, I64, I64, P, P, P, P, P]
        L.relax_q4_matmul_allreduce.restype = I
        _lib = L
        return L


def _check(rc: int, where: str):
    if rc != RELAX_OK:
        raise RelaxError(rc, where)


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def plan_workspace(n_max: int, K: int, N: int) -> int:
    """Bytes of workspace that make every relax_q4_matmul_ws call with n <= n_max succeed."""
    out = ctypes.c_size_t(0)
    _check(lib().relax_plan_workspace(n_max, K, N, ctypes.byref(out)), "relax_plan_workspace")
    return int(out.value)


def query_schedule(n: int, K: int, N: int) -> dict:
    v, t, s, pe = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    ws = ctypes.c_size_t(0)
    _check(lib().relax_query_schedule(n, K, N, ctypes.byref(v), ctypes.byref(t), ctypes.byref(s),
                                      ctypes.byref(ws), ctypes.byref(pe)), "relax_query_schedule")
    name = {VARIANT_GEMV: "gemv", VARIANT_TC: "tc", VARIANT_SMALLN: "smalln"}[v.value]
    d = {"variant": name, "tile": t.value, "split_k": s.value, "ws_bytes": int(ws.value)}
    if pe.value:
        d["persistent"] = True
    if pe.value == 2:
        d["stream_k"] = True
    if pe.value in (3, 4):                 # whole tiles over the leading rows + a split-K launch for the rest
        del d["persistent"]
        d["two_part"] = True
        if pe.value == 4:                  # the leading rows on the persistent kernel
            d["two_part_persistent"] = True
    return d


def _device_of_call():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def _check_tensor(t, name, dtype, shape=None, dev=None):
    """Every tensor crossing the boundary: CUDA, on the current device, dense
    row-major, of the ABI's dtype and (where given) shape.  The C-ABI only sees
    pointers, so a mismatch here would otherwise read or write out of bounds."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype not in (dtype if isinstance(dtype, tuple) else (dtype,)):
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_cuda or (dev is not None and t.device != dev):
        raise ValueError(f"{name}: on {t.device}, expected the current CUDA device {dev}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous (dense row-major)")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")


def _shapes(x, packed_w, scales):
    import torch
    dev = _device_of_call()
    if x.dim() != 2 or packed_w.dim() != 2 or scales.dim() != 2:
        raise ValueError("x, packed_w and scales must be 2-D")
    n, K = x.shape
    N = packed_w.shape[0]
    if packed_w.shape[1] * 8 != K or scales.shape != (N, K // 32):
        raise ValueError(f"shape mismatch: x {tuple(x.shape)} packed_w {tuple(packed_w.shape)} "
                         f"scales {tuple(scales.shape)}")
    _check_tensor(x, "x", torch.float16, dev=dev)
    _check_tensor(packed_w, "packed_w", (torch.int32, torch.uint32), dev=dev)
    _check_tensor(scales, "scales", torch.float16, dev=dev)
    return n, K, N


def _out(y, n, N, x):
    import torch
    if y is None:
        return torch.empty((n, N), dtype=torch.float16, device=x.device)
    _check_tensor(y, "y", torch.float16, (n, N), dev=x.device)
    return y


def _ws_bytes(ws, dev):
    if ws is None:
        return 0
    import torch
    _check_tensor(ws, "ws", (torch.uint8, torch.int8, torch.int32, torch.float32), dev=dev)
    return ws.numel() * ws.element_size()


def workspace(n_max: int, K: int, N: int, device=None):
    """Allocate a zero-filled workspace sized by plan_workspace (None if 0 bytes)."""
    import torch
    nb = plan_workspace(n_max, K, N)
    if nb == 0:
        return None
    return torch.zeros(nb, dtype=torch.uint8, device=device or "cuda")


def q4_matmul(x, packed_w, scales, y=None, ws=None, stream=None):
    """y[n, N] = x[n, K] . dequant(packed_w, scales) via relax_q4_matmul(_ws)."""
    n, K, N = _shapes(x, packed_w, scales)
    y = _out(y, n, N, x)
    nb = _ws_bytes(ws, x.device)
    st = _stream_ptr(stream)
    if ws is None:
        rc = lib().relax_q4_matmul(_ptr(x), n, K, N, _ptr(packed_w), _ptr(scales), _ptr(y), st)
        _check(rc, "relax_q4_matmul")
    else:
        rc = lib().relax_q4_matmul_ws(_ptr(x), n, K, N, _ptr(packed_w), _ptr(scales), _ptr(y),
                                      _ptr(ws), nb, st)
        _check(rc, "relax_q4_matmul_ws")
    return y


def q4_matmul_grouped(x, weights, ys=None, stream=None):
    """relax_q4_matmul_grouped: y_i = x . dequant(packed_w_i, scales_i) for a list
    of (packed_w, scales) pairs sharing x (q/k/v, gate/up): one launch at decode."""
    import torch
    if not 1 <= len(weights) <= 4:
        raise ValueError("1..4 linears per group")
    outs = []
    for i, (pw, sc) in enumerate(weights):
        n, K, N = _shapes(x, pw, sc)
        outs.append(_out(None if ys is None else ys[i], n, N, x))
    cnt = len(weights)
    Ns = (ctypes.c_int64 * cnt)(*[pw.shape[0] for pw, _ in weights])
    Ws = (ctypes.c_void_p * cnt)(*[_ptr(pw) for pw, _ in weights])
    Ss = (ctypes.c_void_p * cnt)(*[_ptr(sc) for _, sc in weights])
    Ys = (ctypes.c_void_p * cnt)(*[_ptr(y) for y in outs])
    rc = lib().relax_q4_matmul_grouped(_ptr(x), x.shape[0], x.shape[1], cnt, Ns, Ws, Ss, Ys, _stream_ptr(stream))
    _check(rc, "relax_q4_matmul_grouped")
    return outs


def has_chain() -> bool:
    """Whether the loaded library is the experiments build with the decode chain."""
    return hasattr(lib(), "relax_q4_chain_run")


class DecodeChain:
    """relax_q4_chain_* (experiments build only; RELAX_Q4_LIB=build_exp/...): a
    fixed sequence of n = 1 matmuls run as ONE persistent launch.  ops: list of (x, packed_w, scales, y, after) with x fp16 [1, K] (or
    [K]), y fp16 [1, N]; `after` = the op reads what an earlier op wrote (it
    waits for every earlier op).  The tensors must stay alive and in place: the
    chain keeps their pointers."""

    def __init__(self, ops, device=None):
        import torch
        if not has_chain():
            raise RelaxError(1, "relax_q4_chain_init (not in this library: build --experiments and set RELAX_Q4_LIB)")
        dev = _device_of_call()
        arr = (ChainOp * len(ops))()
        self._keep = []
        for i, (x, pw, sc, y, after) in enumerate(ops):
            N, K = pw.shape[0], pw.shape[1] * 8
            _check_tensor(x, f"ops[{i}].x", torch.float16, dev=dev)
            _check_tensor(pw, f"ops[{i}].packed_w", (torch.int32, torch.uint32), dev=dev)
            _check_tensor(sc, f"ops[{i}].scales", torch.float16, (N, K // 32), dev=dev)
            _check_tensor(y, f"ops[{i}].y", torch.float16, dev=dev)
            if x.numel() != K or y.numel() != N:
                raise ValueError(f"ops[{i}]: x has {x.numel()} elements (K = {K}), y {y.numel()} (N = {N})")
            arr[i] = ChainOp(_ptr(x), _ptr(pw), _ptr(sc), _ptr(y), K, N, 1 if after else 0, 0)
            self._keep.append((x, pw, sc, y))
        nb = ctypes.c_size_t(0)
        _check(lib().relax_q4_chain_workspace(len(ops), ctypes.byref(nb)), "relax_q4_chain_workspace")
        self.ws = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
        _check(lib().relax_q4_chain_init(arr, len(ops), _ptr(self.ws), int(nb.value)), "relax_q4_chain_init")
        self.count = len(ops)

    def run(self, stream=None):
        _check(lib().relax_q4_chain_run(_ptr(self.ws), _stream_ptr(stream)), "relax_q4_chain_run")


def tp_comm_bytes(world: int, N_max: int) -> int:
    """relax_tp_comm_bytes: exchange-buffer bytes per rank for outputs of <= N_max features."""
    out = ctypes.c_size_t(0)
    _check(lib().relax_tp_comm_bytes(world, N_max, ctypes.byref(out)), "relax_tp_comm_bytes")
    return int(out.value)


def make_tp_comm(world: int, rank: int, buf_ptrs, buf_bytes: int) -> TpComm:
    """The relax_tp_comm of this rank from the ranks' buffer pointers (as
    mapped on this device; e.g. torch symmetric memory's buffer_ptrs)."""
    if not 1 <= world <= TP_MAX_WORLD or not 0 <= rank < world or len(buf_ptrs) != world:
        raise ValueError(f"world {world}, rank {rank}, {len(buf_ptrs)} buffers")
    c = TpComm()
    c.world, c.rank, c.buf_bytes = world, rank, int(buf_bytes)
    for p, ptr in enumerate(buf_ptrs):
        c.bufs[p] = int(ptr)
    return c


def q4_matmul_allreduce(x, packed_w, scales, comm: TpComm, residual=None, y=None, stream=None):
    """relax_q4_matmul_allreduce: y = fp16(sum over ranks of x_r . W_r) (+ residual)
    with the sum fused into the decode kernel over the ranks' exchange buffers
    (n <= 2; every rank must make the same sequence of calls)."""
    import torch
    n, K, N = _shapes(x, packed_w, scales)
    y = _out(y, n, N, x)
    if residual is not None:
        _check_tensor(residual, "residual", torch.float16, (n, N), dev=x.device)
    rc = lib().relax_q4_matmul_allreduce(ctypes.byref(comm), _ptr(x), n, K, N, _ptr(packed_w), _ptr(scales),
                                         _ptr(residual), _ptr(y), _stream_ptr(stream))
    _check(rc, "relax_q4_matmul_allreduce")
    return y


def q4_matmul_ex(x, packed_w, scales, y=None, ws=None, variant=VARIANT_AUTO, split_k=0, bn=0,
                 flags=0, stream=None):
    n, K, N = _shapes(x, packed_w, scales)
    y = _out(y, n, N, x)
    nb = _ws_bytes(ws, x.device)
    rc = lib().relax_q4_matmul_ex(_ptr(x), n, K, N, _ptr(packed_w), _ptr(scales), _ptr(y),
                                  _ptr(ws), nb, variant, split_k, bn, flags, _stream_ptr(stream))
    _check(rc, "relax_q4_matmul_ex")
    return y


def q4_dequant(packed_w, scales, K: int, w_out=None, stream=None):
    """w_out[N, K] fp16 = fp16_RNE((q - 7) * s), bit-exact."""
    import torch
    dev = _device_of_call()
    if packed_w.dim() != 2 or packed_w.shape[1] * 8 != K:
        raise ValueError(f"packed_w {tuple(packed_w.shape)} does not hold K = {K} codes per row")
    N = packed_w.shape[0]
    _check_tensor(packed_w, "packed_w", (torch.int32, torch.uint32), dev=dev)
    _check_tensor(scales, "scales", torch.float16, (N, K // 32), dev=dev)
    if w_out is None:
        w_out = torch.empty((N, K), dtype=torch.float16, device=packed_w.device)
    else:
        _check_tensor(w_out, "w_out", torch.float16, (N, K), dev=dev)
    rc = lib().relax_q4_dequant(_ptr(packed_w), _ptr(scales), K, N, _ptr(w_out), _stream_ptr(stream))
    _check(rc, "relax_q4_dequant")
    return w_out


def plan_workspace_fused(n_max: int, K: int, N: int, ops: int) -> int:
    out = ctypes.c_size_t(0)
    _check(lib().relax_plan_workspace_fused(n_max, K, N, ops, ctypes.byref(out)), "relax_plan_workspace_fused")
    return int(out.value)


def q4_matmul_fused(x, packed_w, scales, y=None, rms_weight=None, rms_eps: float = 1e-5, silu_mul: bool = False,
                    residual=None, kv_append=None, ws=None, stream=None):
    """relax_q4_matmul_fused: optional RMSNorm prologue on x (rms_weight = gamma [K]),
    SiLU-mul epilogue over interleaved (gate, up) rows (y has N/2 columns), a
    residual add, and (decode) the KV append: kv_append = (k_cache, v_cache,
    pos, row0) stores y's rows row0 .. row0 + 2 H 128 (keys, then values) at
    cache position pos[t]; see include/relax_q4.h for the exact semantics."""
    import torch
    n, K, N = _shapes(x, packed_w, scales)
    ops = (OP_RMSNORM_X if rms_weight is not None else 0) | (OP_SILU_MUL if silu_mul else 0) | \
          (OP_RESIDUAL if residual is not None else 0) | (OP_KV_APPEND if kv_append is not None else 0)
    n_out = N // 2 if silu_mul else N
    y = _out(y, n, n_out, x)
    if rms_weight is not None:
        _check_tensor(rms_weight, "rms_weight", torch.float16, (K,), dev=x.device)
    if residual is not None:
        _check_tensor(residual, "residual", torch.float16, (n, n_out), dev=x.device)
    fz = Fusion(ops, float(rms_eps), _ptr(rms_weight) or None, _ptr(residual) or None)
    if kv_append is not None:
        kc, vc, pos, row0 = kv_append
        if kc.dim() != 4 or kc.shape[0] != n or kc.shape[3] != 128:
            raise ValueError(f"k_cache: shape {tuple(kc.shape)}, expected [n, H, L_max, 128]")
        _check_tensor(kc, "k_cache", torch.float16, dev=x.device)
        _check_tensor(vc, "v_cache", torch.float16, tuple(kc.shape), dev=x.device)
        _check_tensor(pos, "pos", torch.int32, (n,), dev=x.device)
        fz.k_cache, fz.v_cache, fz.kv_pos = _ptr(kc), _ptr(vc), _ptr(pos)
        fz.kv_len_max, fz.kv_heads, fz.kv_row0 = kc.shape[2], kc.shape[1], int(row0)
    nb = _ws_bytes(ws, x.device)
    rc = lib().relax_q4_matmul_fused(_ptr(x), n, K, N, _ptr(packed_w), _ptr(scales), _ptr(y), ctypes.byref(fz),
                                     _ptr(ws), nb, _stream_ptr(stream))
    _check(rc, "relax_q4_matmul_fused")
    return y


def attn_decode_workspace(batch: int, n_heads: int, kv_len_max: int) -> int:
    out = ctypes.c_size_t(0)
    _check(lib().relax_attn_decode_workspace(batch, n_heads, kv_len_max, ctypes.byref(out)),
           "relax_attn_decode_workspace")
    return int(out.value)


def attn_decode(q, k_cache, v_cache, kv_lens, out=None, ws=None, stream=None):
    """relax_attn_decode: q [batch, Hq, 128] fp16, caches [batch, Hkv, L_max, 128]
    fp16, kv_lens int32 [batch] (device) -> out [batch, Hq, 128] fp16."""
    import torch
    dev = _device_of_call()
    if q.dim() != 3 or k_cache.dim() != 4:
        raise ValueError("q must be [batch, Hq, D] and the caches [batch, Hkv, L_max, D]")
    batch, hq, d = q.shape
    _, hkv, lmax, _ = k_cache.shape
    _check_tensor(q, "q", torch.float16, dev=dev)
    _check_tensor(k_cache, "k_cache", torch.float16, (batch, hkv, lmax, d), dev=dev)
    _check_tensor(v_cache, "v_cache", torch.float16, (batch, hkv, lmax, d), dev=dev)
    _check_tensor(kv_lens, "kv_lens", torch.int32, (batch,), dev=dev)
    out = _out(out.view(batch, hq * d) if out is not None else None, batch, hq * d, q).view(batch, hq, d)
    if ws is None:
        nb = attn_decode_workspace(batch, hq, lmax)
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)
    nb = _ws_bytes(ws, dev)
    rc = lib().relax_attn_decode(_ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(kv_lens), batch, hq, hkv, d, lmax,
                                 _ptr(out), _ptr(ws), nb, _stream_ptr(stream))
    _check(rc, "relax_attn_decode")
    return out


def kv_append(k_new, v_new, pos, k_cache, v_cache, stream=None):
    """relax_kv_append: write k_new, v_new [batch, Hkv, 128] at pos[b] of each cache."""
    import torch
    dev = _device_of_call()
    batch, hkv, lmax, d = k_cache.shape
    _check_tensor(k_new, "k_new", torch.float16, (batch, hkv, d), dev=dev)
    _check_tensor(v_new, "v_new", torch.float16, (batch, hkv, d), dev=dev)
    _check_tensor(pos, "pos", torch.int32, (batch,), dev=dev)
    _check_tensor(k_cache, "k_cache", torch.float16, dev=dev)
    _check_tensor(v_cache, "v_cache", torch.float16, (batch, hkv, lmax, d), dev=dev)
    rc = lib().relax_kv_append(_ptr(k_new), _ptr(v_new), _ptr(pos), batch, hkv, d, lmax, _ptr(k_cache),
                               _ptr(v_cache), _stream_ptr(stream))
    _check(rc, "relax_kv_append")


LAYOUT_NK, LAYOUT_KN, LAYOUT_NK3 = 0, 1, 2


def q4_repack(src_packed, src_scales, K: int, N: int, layout: str = "kn", group: int = 32,
              packed_w=None, scales=None, stream=None):
    """relax_q4_repack: convert a weight stored as `layout` ("nk" / "kn" / "nk3" = 3-bit) with
    group size `group` into the native packed_w [N, K/8] (int32) and scales
    [N, K/32] (fp16); bit-exact (include/relax_q4.h)."""
    import torch
    lay = {"nk": LAYOUT_NK, "kn": LAYOUT_KN, "nk3": LAYOUT_NK3}[layout]
    dev = _device_of_call()
    if K % group != 0 or group not in (32, 64, 128):
        raise ValueError(f"group {group} must be 32, 64 or 128 and divide K = {K}")
    want_p = {LAYOUT_NK: (N, K // 8), LAYOUT_KN: (K // 8, N), LAYOUT_NK3: (N, K // 32 * 3)}[lay]
    want_s = (K // group, N) if lay == LAYOUT_KN else (N, K // group)
    _check_tensor(src_packed, "src_packed", (torch.int32, torch.uint32), want_p, dev=dev)
    _check_tensor(src_scales, "src_scales", torch.float16, want_s, dev=dev)
    if packed_w is None:
        packed_w = torch.empty((N, K // 8), dtype=torch.int32, device=dev)
    else:
        _check_tensor(packed_w, "packed_w", (torch.int32, torch.uint32), (N, K // 8), dev=dev)
    if scales is None:
        scales = torch.empty((N, K // 32), dtype=torch.float16, device=dev)
    else:
        _check_tensor(scales, "scales", torch.float16, (N, K // 32), dev=dev)
    rc = lib().relax_q4_repack(_ptr(src_packed), _ptr(src_scales), K, N, lay, group, _ptr(packed_w),
                               _ptr(scales), _stream_ptr(stream))
    _check(rc, "relax_q4_repack")
    return packed_w, scales


def interleave_rows(a, b):
    """Weight prep for the SiLU-mul epilogue (a one-time repack): rows of a
    (gate) and b (up) alternated, out[2j] = a[j], out[2j+1] = b[j]."""
    import torch
    if a.shape != b.shape:
        raise ValueError("gate and up must have the same shape")
    return torch.stack((a, b), dim=1).reshape((2 * a.shape[0],) + tuple(a.shape[1:])).contiguous()


def version() -> str:
    return lib().relax_version().decode()
