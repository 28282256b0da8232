"""Tensor-parallel sharding of q4f16 linears over torch.distributed.

One process per GPU; the data path per rank is the C-ABI kernel
(relax_q4_matmul) on the rank's shard, and the only exchange is one NCCL
collective where the sharding needs one (NVLink 5 / NVSwitch on the box):

  column split (N/p rows of the NK layout per rank, contiguous -- no repack):
      y_r[n, N/p] = x[n, K] . W_r            ; optional all_gather -> y[n, N]
  row split    (K/p slice of every row, materialised once at load time):
      y_r[n, N]   = x_r[n, K/p] . W_r        ; all_reduce(sum) -> y[n, N]

Megatron pairing for a Llama decoder block: q/k/v and gate/up column-split
feed o and down row-split, one all_reduce after each (2 per layer).

The per-rank matmul is injectable (`matmul`) so the host-side sharding and
collective logic can be tested on CPU with the gloo backend; the product path
uses ops.q4_matmul and has no fallback.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

GROUP = 32


def shard_bounds(total: int, rank: int, world: int, align: int = 1):
    """[lo, hi) of `total` for `rank`, split into `world` equal aligned parts."""
    if total % (world * align) != 0:
        raise ValueError(f"{total} not divisible into {world} parts aligned to {align}")
    part = total // world
    return rank * part, (rank + 1) * part


def shard_columns(packed, scales, rank: int, world: int):
    """Column split: output features [N r/p, N (r+1)/p) -- contiguous rows of
    packed_w [N][K/8] and scales [N][K/32]."""
    N = packed.shape[0]
    lo, hi = shard_bounds(N, rank, world)
    return packed[lo:hi], scales[lo:hi]


def shard_rows(packed, scales, rank: int, world: int):
    """Row split: reduction range k in [K r/p, K (r+1)/p); K/p must be a
    multiple of the 32-code group (and of 256 for the tensor-core variant)."""
    K = packed.shape[1] * 8
    lo, hi = shard_bounds(K, rank, world, GROUP)
    pk = packed[:, lo // 8:hi // 8]
    sc = scales[:, lo // GROUP:hi // GROUP]
    # materialise contiguous shards (done once, at weight-load time)
    if hasattr(pk, "contiguous"):
        return pk.contiguous(), sc.contiguous()
    return np.ascontiguousarray(pk), np.ascontiguousarray(sc)


def _default_matmul():
    from . import ops
    return lambda x, pk, sc: ops.q4_matmul(x, pk, sc)


@dataclass
class ColumnParallelQ4:
    """y_r = x . W_r on this rank's N/p output features; with gather=True the
    shards are all-gathered (NCCL all_gather_into_tensor over NVLink on the
    box) into the full [n, N] in feature order -- the lm_head's logits."""
    packed: object
    scales: object
    group: object = None
    gather: bool = False
    matmul: Optional[Callable] = None

    def __call__(self, x):
        import torch
        import torch.distributed as dist
        mm = self.matmul or _default_matmul()
        y = mm(x, self.packed, self.scales)               # [n, N/p]
        if not self.gather:
            return y
        world = dist.get_world_size(self.group)
        n, npart = y.shape
        buf = torch.empty((world * n, npart), dtype=y.dtype, device=y.device)
        dist.all_gather_into_tensor(buf, y.contiguous(), group=self.group)
        # [p*n][N/p] = [p][n][N/p] -> [n][N]: rank r's features are columns [r N/p, (r+1) N/p)
        return buf.view(world, n, npart).permute(1, 0, 2).reshape(n, world * npart)


class TpExchange:
    """The exchange buffers of relax_q4_matmul_allreduce (the row split with
    its all-reduce fused into the decode kernel) for one
    process group.  torch symmetric memory is the plumbing: it allocates each
    rank's buffer and maps every peer's buffer into this process (NVLink peer
    memory on the box); the library only sees the pointers.  The buffers are
    zero-filled and the group synchronised once here; afterwards every rank
    must issue the same sequence of fused calls (include/relax_q4.h)."""

    def __init__(self, N_max: int, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        from . import ops
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.N_max = N_max
        self.nbytes = ops.tp_comm_bytes(self.world, N_max)
        self.buf = symm.empty(self.nbytes, dtype=torch.uint8, device=torch.device("cuda", torch.cuda.current_device()))
        name = (group if group is not None else dist.group.WORLD).group_name
        self.handle = symm.rendezvous(self.buf, name)
        ptrs = list(self.handle.buffer_ptrs)
        off = self.buf.data_ptr() - ptrs[self.rank]          # the same offset in every rank's allocation
        self.buf.zero_()
        torch.cuda.synchronize()
        dist.barrier(group=group)
        self.comm = ops.make_tp_comm(self.world, self.rank, [p + off for p in ptrs], self.nbytes)


def fused_allreduce_ok(n: int, K: int) -> bool:
    """Whether relax_q4_matmul_allreduce takes this call (decode n <= 2, K % 256 == 0)."""
    return 1 <= n <= 2 and K % 256 == 0


@dataclass
class RowParallelQ4:
    """Partial y_r = x_r . W_r over this rank's K/p slice, summed over the
    ranks.  With an `exchange` (TpExchange) and a decode-sized x, the sum is
    fused into the kernel (relax_q4_matmul_allreduce: fp32 partials over
    NVLink peer memory, summed in rank order, one fp16 rounding).  Otherwise
    one NCCL all_reduce: the kernel's partials are fp16 (its output type), the
    sum runs in fp32 and is rounded to fp16 once (DESIGN.md §3 reading 14)."""
    packed: object
    scales: object
    group: object = None
    matmul: Optional[Callable] = None
    reduce_fp32: bool = True
    exchange: Optional[TpExchange] = None
    stream: object = None

    def __call__(self, x_shard):
        import torch
        import torch.distributed as dist
        if self.exchange is not None and fused_allreduce_ok(x_shard.shape[0], x_shard.shape[1]):
            from . import ops
            return ops.q4_matmul_allreduce(x_shard, self.packed, self.scales, self.exchange.comm,
                                           stream=self.stream)
        mm = self.matmul or _default_matmul()
        y = mm(x_shard, self.packed, self.scales)         # partial [n, N]
        if self.reduce_fp32:
            y32 = y.float()
            dist.all_reduce(y32, op=dist.ReduceOp.SUM, group=self.group)
            return y32.to(torch.float16)
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y


# Megatron placement of the Llama linears: column-parallel
# producers, row-parallel consumers, one all_reduce after each row-parallel
# linear; the lm_head column-parallel with its logits gathered.
MEGATRON_KIND = {"q": "col", "k": "col", "v": "col", "qkv": "col", "gate": "col", "up": "col",
                 "gate_up": "col", "o": "row", "down": "row", "lm_head": "col"}


def shard_shape(name: str, K: int, N: int, world: int):
    """Rank-local (K, N) of a linear under Megatron TP of degree `world`."""
    if world == 1:
        return K, N
    if MEGATRON_KIND[name] == "row":
        lo, hi = shard_bounds(K, 0, world, GROUP)
        return hi - lo, N
    lo, hi = shard_bounds(N, 0, world)
    return K, hi - lo


def megatron_linear(name: str, packed, scales, group=None, matmul=None, exchange=None, stream=None):
    """The TP wrapper of one Llama linear given this rank's shard (`exchange`:
    the row-split linears fuse their all-reduce at decode)."""
    if MEGATRON_KIND[name] == "row":
        return RowParallelQ4(packed, scales, group=group, matmul=matmul, exchange=exchange, stream=stream)
    return ColumnParallelQ4(packed, scales, group=group, gather=(name == "lm_head"), matmul=matmul)


def split_x_for_rows(x, rank: int, world: int):
    """The K-slice of x a row-split rank consumes."""
    K = x.shape[1]
    lo, hi = shard_bounds(K, rank, world, GROUP)
    xs = x[:, lo:hi]
    return xs.contiguous() if hasattr(xs, "contiguous") else np.ascontiguousarray(xs)
