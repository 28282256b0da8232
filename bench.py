#!/usr/bin/env python3
"""bench.py -- Llama-2 layer-set throughput of the fused q4f16 dequant-matmul.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload llama2-7b-decode|llama2-13b-decode|llama2-70b-decode|llama2-7b-prefill|...]
                    [--n TOKENS] [--fused] [--replicas] [--tp-shard P] [--block fused|unfused]

A step = one pass of the whole hot path over one batch: every linear layer of
the model (32 x {q,k,v,o,gate,up,down} + lm_head for 7B) applied to n tokens,
each a relax_q4_matmul call (weights resident in HBM, distinct buffers per
layer, so the 3.7 GB working set streams from HBM -- far larger than the
126 MB L2, no flush needed).  The step is captured once into a CUDA graph
(programmatic dependent launch between consecutive kernels) and replayed.

Default workload = BASELINE.json config 2, "Llama-2-7B decode weight set at
n=1 on 1 B200"; value = tokens/s.

--gpus N (N > 1): re-launches itself under torch.distributed.run (one rank per
GPU, NCCL, 127.0.0.1) unless already under torchrun.  With N > 1 ranks the
default is Megatron tensor parallelism of the layer set (north_star item 3,
SURVEY §8(e)): q/k/v and gate/up stacked and column-split, o and down
row-split with an fp32 all_reduce of the partial y, the lm_head column-split
with its logits all-gathered -- paper_2311_02103_b200/tp.py, the code the
gloo and NCCL tests check; one token stream, "scaling": "strong".
--replicas instead runs N independent decode replicas (no collective,
"scaling": "weak").

--impl reference times the CPU oracle (oracle/, the only reference that
exists: the paper ships no code) on the host cores, same metric and config;
each step is a bounded sample (one linear of layer 0, full outputs, rotating
through the seven; extrapolated by multiply-accumulate count to the layer set).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2311_02103_b200 import inputs  # noqa: E402  (seeded generators only)

METRIC = BASELINE_METRIC = ("q4 dequant-matmul HBM GB/s (n=1) & TFLOPS (n≥512); "
                            "Llama-2 layer-set tok/s")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "src": "fallback"}


# (query heads, kv heads) of each model; head_dim 128
HEADS = {"llama2-7b": (32, 32), "llama2-13b": (40, 40), "llama2-70b": (64, 8)}


def layer_set(workload: str, fused: bool = False, tp: int = 1):
    """The linears of one token.  fused=True stacks the rows of q/k/v and of
    gate/up (the NK layout makes that a concatenation) into one call each --
    same weights, same bytes, 4 dependent calls per layer instead of 7.
    tp=p gives the rank-local shard shapes of a p-way Megatron split
    (tp.shard_shape: column-parallel q/k/v, gate/up, lm_head; row-parallel
    o, down)."""
    from paper_2311_02103_b200 import tp as tpm
    model = workload.rsplit("-", 1)[0]          # llama2-7b-decode -> llama2-7b
    spec = inputs.LLAMA_SETS[model]
    mats = []
    for li in range(spec["layers"]):
        if fused:
            d = {name: (K, N) for name, K, N in spec["mats"]}
            K = d["q"][0]
            layer = [("qkv", K, d["q"][1] + d["k"][1] + d["v"][1]), ("o", *d["o"]),
                     ("gate_up", K, d["gate"][1] + d["up"][1]), ("down", *d["down"])]
        else:
            layer = list(spec["mats"])
        for name, K, N in layer:
            mats.append((f"L{li}.{name}", *tpm.shard_shape(name, K, N, tp)))
    mats.append(("lm_head", *tpm.shard_shape("lm_head", *spec["lm_head"], tp)))
    return model, mats


def algorithmic(mats, n):
    """Algorithmic bytes (weights once, x once, y once) and flops per step."""
    b = sum(inputs.q4_bytes(K, N) + 2 * n * K + 2 * n * N for _, K, N in mats)
    f = sum(2 * n * K * N for _, K, N in mats)
    return b, f


# --------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


# --------------------------------------------------------------------- ours
def block_step(args, mats, weights, n, dev, stream):
    """Decoder-block chain over the fused-layout linears:
    per layer  qkv = W_qkv . RMSNorm(h);  h += W_o . a;  act = SiLU(g) * u with
    [g; u] = W_gate_up . RMSNorm(h);  h += W_down . act;  then logits =
    W_head . RMSNorm(h).  Without --kv the attention is a fixed fp16 tensor `a`
    standing in for its output; with --kv L (fused block, n = 1) it is the
    library's decode attention: the new token's k, v (slices
    of the qkv output) stored at position L - 1 of the layer's fp16 KV cache by
    the qkv kernel itself (RELAX_OP_KV_APPEND epilogue) and q attending over the L cached keys
    (relax_attn_decode) -- the whole decode step, attention over a symbolic KV
    length included (RoPE is not applied: it does not change what is read or
    computed per byte).  --block fused runs each linear
    with its neighbours fused (relax_q4_matmul_fused: 4 kernels per layer,
    gate/up rows interleaved); --block unfused runs the same linears through
    relax_q4_matmul with the element-wise ops as separate torch kernels (the
    unfused program: our matmuls + torch eager glue, not launched with PDL)."""
    import torch
    from paper_2311_02103_b200 import ops
    model = args.workload.rsplit("-", 1)[0]
    hidden = inputs.LLAMA_SETS[model]["mats"][0][1]
    hq, hkv = HEADS[model]
    kv = None
    if args.kv > 0:
        if args.block != "fused" or n != 1:
            raise SystemExit("--kv needs --block fused at n = 1 (the qkv output slices are the new q, k, v)")
        L = args.kv
        g = torch.Generator(device=dev)
        g.manual_seed(11)
        nl = sum(1 for nm, _, _ in mats if nm.endswith(".qkv"))
        kv = {"k": [torch.randn((1, hkv, L, 128), generator=g, device=dev).half() for _ in range(nl)],
              "v": [torch.randn((1, hkv, L, 128), generator=g, device=dev).half() for _ in range(nl)],
              "lens": torch.tensor([L], dtype=torch.int32, device=dev),
              "pos": torch.tensor([L - 1], dtype=torch.int32, device=dev),
              "out": torch.empty((1, hq, 128), dtype=torch.float16, device=dev)}
        kv["ws"] = torch.empty(ops.attn_decode_workspace(1, hq, L), dtype=torch.uint8, device=dev)
    h0 = torch.from_numpy(inputs.activations(3, n, hidden).view(np.float16)).to(dev)
    h = h0.clone()
    attn = torch.from_numpy(inputs.activations(4, n, hidden).view(np.float16)).to(dev)
    gamma = torch.from_numpy((np.random.default_rng(5).uniform(0.8, 1.2, hidden)).astype(np.float16)).to(dev)
    eps = 1e-5
    outs = {}
    for (name, K, N) in mats:
        kind = name.split(".")[-1]
        if kind == "gate_up":
            outs[name] = torch.empty((n, N // 2 if args.block == "fused" else N), dtype=torch.float16, device=dev)
        elif kind in ("qkv", "lm_head"):
            outs[name] = torch.empty((n, N), dtype=torch.float16, device=dev)
    tmp = torch.empty((n, hidden), dtype=torch.float16, device=dev)
    wss = {}
    for (name, K, N) in mats:
        nb = ops.plan_workspace_fused(n, K, N, ops.OP_RMSNORM_X | (ops.OP_SILU_MUL if "gate_up" in name else 0))
        wss[name] = torch.zeros(nb, dtype=torch.uint8, device=dev) if nb else None

    def rms(v):
        vf = v.float()
        r = torch.rsqrt(vf.pow(2).mean(-1, keepdim=True) + eps)
        return (vf * r).half() * gamma

    def step():
        h.copy_(h0)                                      # every step decodes the same token
        act = None
        li = 0
        for (name, K, N), (pk, sc) in zip(mats, weights):
            kind = name.split(".")[-1]
            if args.block == "fused":
                if kind in ("qkv", "lm_head"):
                    # with the KV cache the new token's k, v go to their cache
                    # position in the same kernel (RELAX_OP_KV_APPEND epilogue)
                    kva = (kv["k"][li], kv["v"][li], kv["pos"], hq * 128) if kind == "qkv" and kv is not None else None
                    ops.q4_matmul_fused(h, pk, sc, y=outs[name], rms_weight=gamma, rms_eps=eps, ws=wss[name],
                                        kv_append=kva, stream=stream)
                    if kind == "qkv" and kv is not None:
                        y = outs[name]
                        qv = y[:, :hq * 128].view(1, hq, 128)
                        ops.attn_decode(qv, kv["k"][li], kv["v"][li], kv["lens"], out=kv["out"], ws=kv["ws"],
                                        stream=stream)
                        li += 1
                elif kind == "o":
                    a_in = attn if kv is None else kv["out"].view(1, hq * 128)
                    ops.q4_matmul_fused(a_in, pk, sc, y=h, residual=h, stream=stream)
                elif kind == "gate_up":
                    act = outs[name]
                    ops.q4_matmul_fused(h, pk, sc, y=act, rms_weight=gamma, rms_eps=eps, silu_mul=True,
                                        ws=wss[name], stream=stream)
                else:                                    # down
                    ops.q4_matmul_fused(act, pk, sc, y=h, residual=h, stream=stream)
            else:
                if kind in ("qkv", "lm_head"):
                    ops.q4_matmul(rms(h), pk, sc, y=outs[name], stream=stream)
                elif kind == "o":
                    ops.q4_matmul(attn, pk, sc, y=tmp, stream=stream)
                    h.add_(tmp)
                elif kind == "gate_up":
                    gu = outs[name]
                    ops.q4_matmul(rms(h), pk, sc, y=gu, stream=stream)
                    act = torch.nn.functional.silu(gu[:, 0::2]) * gu[:, 1::2]
                else:
                    ops.q4_matmul(act.contiguous(), pk, sc, y=tmp, stream=stream)
                    h.add_(tmp)
    return step, (h0, outs[mats[-1][0]])


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2311_02103_b200 import ops
    from paper_2311_02103_b200 import tp as tpm

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    ops.lib()
    tp_mode = args.tp and dist.is_initialized()
    tp_world = world if tp_mode else 1
    if tp_mode and args.tp_shard > 1:
        raise SystemExit("tensor parallelism over the ranks and --tp-shard are exclusive")
    if tp_mode and args.block != "none":
        raise SystemExit("--block runs on one GPU (or as --replicas)")
    # TP runs the Megatron layout: q/k/v and gate/up stacked, as Megatron does
    fused = args.fused or tp_mode
    model, mats = layer_set(args.workload, fused, tp_world if tp_mode else args.tp_shard)
    n = args.n
    t_gen = time.time()
    # One realistic weight per distinct shape (seed 1000*config + index; each
    # TP rank its own shard values), copied into a distinct HBM buffer per layer.
    cfg_id = {"llama2-7b": 2, "llama2-13b": 4, "llama2-70b": 5}[model]
    shapes = sorted({(K, N) for _, K, N in mats})
    proto = {}
    for i, (K, N) in enumerate(shapes):
        pk, sc = inputs.realistic_weights(1000 * cfg_id + i + 100 * (rank if tp_mode else 0), K, N)
        proto[(K, N)] = (torch.from_numpy(pk.view(np.int32)).to(dev),
                         torch.from_numpy(sc.view(np.float16)).to(dev))
    weights = []
    for name, K, N in mats:
        pk, sc = proto[(K, N)]
        weights.append((pk.clone(), sc.clone()))
    del proto
    xs = {K: torch.from_numpy(inputs.activations(7 + n + K, n, K).view(np.float16)).to(dev)
          for K in sorted({K for _, K, _ in mats})}
    ys = [torch.empty((n, N), dtype=torch.float16, device=dev) for _, _, N in mats]
    wss = {}
    for _, K, N in mats:
        if (K, N) not in wss:
            nb = ops.plan_workspace(n, K, N)
            wss[(K, N)] = torch.zeros(nb, dtype=torch.uint8, device=dev) if nb else None
    t_gen = time.time() - t_gen
    sched = {f"{K}x{N}": ops.query_schedule(n, K, N) for K, N in shapes}

    stream = torch.cuda.Stream(device=dev)
    flags = ops.FLAG_NO_PDL if args.no_pdl else 0

    def serial_step():
        for (name, K, N), (pk, sc), y in zip(mats, weights, ys):
            ops.q4_matmul_ex(xs[K], pk, sc, y=y, ws=wss[(K, N)], flags=flags, stream=stream)

    # The linears that read the same x in a Llama layer -- q, k, v and gate, up --
    # go out as one relax_q4_matmul_grouped call each (one launch at decode), the
    # others one call each: the layer's true dependency chain (qkv -> o ->
    # gate/up -> down), on the same per-matrix weight buffers.  --serial makes
    # every linear its own dependent call (round 1's schedule).
    groups = []
    i = 0
    while i < len(mats):
        kind = mats[i][0].split(".")[-1]
        span = 3 if kind == "q" else 2 if kind == "gate" else 1
        groups.append(list(range(i, i + span)))
        i += span
    # (a group is one launch at decode, n <= 2, and for small batches, n <= 8;
    # beyond that its members run one by one anyway, so the plain chain is used)
    grouped = not args.serial and not args.no_pdl and n <= 8 and any(len(g) > 1 for g in groups)

    def grouped_step():
        for g in groups:
            if len(g) == 1:
                j = g[0]
                ops.q4_matmul_ex(xs[mats[j][1]], *weights[j], y=ys[j], ws=wss[(mats[j][1], mats[j][2])],
                                 flags=flags, stream=stream)
            else:
                ops.q4_matmul_grouped(xs[mats[g[0]][1]], [weights[j] for j in g], ys=[ys[j] for j in g],
                                      stream=stream)

    # --chain: the whole layer set as ONE persistent launch (relax_q4_chain_run):
    # the same linears and weights, every op after the first of its group waiting
    # for all earlier ops (the layer's dependency chain)
    chain = None
    if args.chain:
        if n != 1 or tp_mode or args.block != "none":
            raise SystemExit("--chain runs the n = 1 layer set on one GPU")
        first_of_group = {g[0] for g in groups} if not args.serial else set(range(len(mats)))
        chain = ops.DecodeChain([(xs[K], *weights[j], ys[j], j in first_of_group)
                                 for j, (name, K, N) in enumerate(mats)])

    def chain_step():
        chain.run(stream=stream)

    step = chain_step if chain is not None else grouped_step if grouped else serial_step
    out_last = lambda: ys[-1]          # noqa: E731  the step's result (logits)
    tp_allreduce = None
    block_io = None
    if args.block != "none":
        step, block_io = block_step(args, mats, weights, n, dev, stream)
    elif tp_mode:
        # Megatron TP over the NCCL group through tp.py -- the
        # code tests/test_tp_gloo.py and tests/test_gpu_tp.py check: column-
        # parallel qkv / gate_up (no exchange), row-parallel o / down (fp32
        # all_reduce of the fp16 partials, reading 14), column-parallel
        # lm_head with its logits all-gathered to [n, vocab].
        def mm_for(K, N):
            ws = wss[(K, N)]
            return lambda x, pk, sc: ops.q4_matmul_ex(x, pk, sc, ws=ws, flags=flags, stream=stream)

        # decode: the row-parallel o / down sum fused into the kernel's
        # epilogue over the ranks' exchange buffers (relax_q4_matmul_allreduce,
        # SURVEY §8(f) F1) unless --nccl-allreduce
        row_N = [N for name, K, N in mats if tpm.MEGATRON_KIND[name.split(".")[-1]] == "row"
                 and tpm.fused_allreduce_ok(n, K)]
        exchange, tp_allreduce = None, "nccl"
        if row_N and not args.nccl_allreduce:
            try:
                exchange = tpm.TpExchange(max(row_N))
                tp_allreduce = "fused-epilogue"
            except Exception as e:  # noqa: BLE001  no peer mapping on this box: the NCCL all_reduce (GPU) instead
                print(f"bench: fused all-reduce unavailable ({type(e).__name__}: {e}); using NCCL", file=sys.stderr)
            # every rank must take the same path
            ok = torch.tensor([1 if exchange is not None else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                exchange, tp_allreduce = None, "nccl (fused exchange unavailable)"
        lin = [tpm.megatron_linear(name.split(".")[-1], pk, sc, matmul=mm_for(K, N), exchange=exchange,
                                   stream=stream)
               for (name, K, N), (pk, sc) in zip(mats, weights)]
        tp_out = [None]

        def step():
            with torch.cuda.stream(stream):
                for (name, K, N), f in zip(mats, lin):
                    tp_out[0] = f(xs[K])

        out_last = lambda: tp_out[0]   # noqa: E731

    # capture the step
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        step()                                  # eager warm-up (kernel attributes, maps)
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()

    def replay():
        if graph is not None:
            graph.replay()
        else:
            with torch.cuda.stream(stream):
                step()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local_rank)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            replay()
        e1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    if world > 1:
        dist.barrier()
    serial_line = None
    if grouped and block_io is None and not tp_mode:
        # the same layer set with every linear its own dependent call, for reference
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=stream):
            serial_step()
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                g2.replay()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                g2.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        ms_s = max_over_ranks(e0.elapsed_time(e1))
        serial_line = {"value": round((world * n * args.steps) / (ms_s / 1e3), 2), "unit": "tok/s",
                       "ms_per_step": round(ms_s / args.steps, 5), "launch_chain": len(mats),
                       "how": "every linear its own dependent relax_q4_matmul call (q, k, v, gate, up not grouped)"}

    # ---- end to end through the public API: pinned host x in, logits out,
    # (a) replaying the captured step, (b) eagerly -- every C-ABI call
    # dispatched from Python each step (binding + host dispatch included).
    x_host = torch.from_numpy(inputs.activations(99, n, mats[0][1]).view(np.float16)).pin_memory()
    x_dev = xs[mats[0][1]] if block_io is None else block_io[0]
    y_last = out_last() if block_io is None else block_io[1]
    out_host = torch.empty(y_last.shape, dtype=torch.float16).pin_memory()

    def e2e_run(fn, steps):
        with torch.cuda.stream(stream):
            for _ in range(2):
                x_dev.copy_(x_host, non_blocking=True)
                fn()
                out_host.copy_(out_last() if block_io is None else block_io[1], non_blocking=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                x_dev.copy_(x_host, non_blocking=True)
                fn()
                out_host.copy_(out_last() if block_io is None else block_io[1], non_blocking=True)
            e1.record(stream)
        t_host = time.perf_counter() - t0
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1)), t_host

    ms_e2e, _ = e2e_run(replay, args.steps)

    def eager_step():
        with torch.cuda.stream(stream):
            step()

    ms_eager, host_eager_s = e2e_run(eager_step, args.steps)

    bytes_step, flops_step = algorithmic(mats, n)
    if args.kv > 0:
        # attention per layer: read L keys and values, append one of each (fp16, head_dim 128)
        hq, hkv = HEADS[model]
        nl = sum(1 for nm, _, _ in mats if nm.endswith(".qkv"))
        bytes_step += nl * (2 * args.kv * hkv * 128 * 2 + 2 * hkv * 128 * 2 + 2 * hq * 128 * 2)
        flops_step += nl * (4 * args.kv * hq * 128)
    ms_step = ms / args.steps
    streams = 1 if tp_mode else world            # TP: the ranks decode one stream together
    tok_s = streams * n * args.steps / (ms / 1e3)
    gbs = bytes_step / (ms_step / 1e3) / 1e9      # per GPU (each rank streams its own shards)
    tflops = flops_step / (ms_step / 1e3) / 1e12
    peaks = load_peaks()
    tc = n >= 128
    if tc:
        roof = {"bound": "tensor", "achieved": round(tflops, 2), "peak": peaks["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": round(tflops / peaks["bf16_tflops_sustained"], 4),
                "peak_src": f"{peaks['src']} bf16 sustained (fp16 dense = bf16 rate)"}
    else:
        roof = {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / peaks["hbm_gbs"], 4), "peak_src": f"{peaks['src']} hbm copy"}
    per_kind = {"tc": lambda: 1, "smalln": lambda: -(-n // 8), "gemv": lambda: -(-n // 2)}
    launches = 0
    for g in ([] if chain is not None else groups if grouped else [[j] for j in range(len(mats))]):
        kinds = [sched[f"{mats[j][1]}x{mats[j][2]}"]["variant"] for j in g]
        if len(g) > 1 and n <= 2:
            launches += -(-n // 2)                     # one grouped decode launch per token pair
        elif len(g) > 1 and n <= 8:
            launches += 1                              # one grouped small-batch launch
        else:
            launches += sum(per_kind[k]() for k in kinds)
    if chain is not None:
        launches = 1
    if args.kv > 0:
        launches += 2 * sum(1 for nm, _, _ in mats if nm.endswith(".qkv"))   # attention partial + combine
    label = (args.workload + ("-fused-qkv-gateup" if fused else "")
             + (f"-tp{args.tp_shard}-rank0-shard" if args.tp_shard > 1 else "")
             + (f"-megatron-tp{tp_world}" if tp_mode else "")
             + (f"-block-{args.block}" if args.block != "none" else "")
             + (f"-attn-kv{args.kv}" if args.kv > 0 else "")
             + ("-chain" if chain is not None else "-grouped-qkv-gateup" if grouped else ""))
    roof["traffic"] = traffic_per_launch(label, n)
    if chain is not None:
        roof["algorithmic_bytes_per_launch"] = int(bytes_step)
        roof["kernel"] = "q4_decode_chain_kernel (the whole layer set in one persistent launch)"
        roof["per"] = "one launch per step"
    else:
        # per launch of the linears (a grouped q/k/v or gate/up launch counts once)
        lin_launches = launches - (2 * sum(1 for nm, _, _ in mats if nm.endswith(".qkv")) if args.kv > 0 else 0)
        roof["algorithmic_bytes_per_launch"] = int(bytes_step / max(lin_launches, 1))
        kind0 = sched[f"{shapes[0][0]}x{shapes[0][1]}"]["variant"]
        roof["kernel"] = {"gemv": "q4_decode_stream_kernel (streamed decode GEMV)",
                          "smalln": "q4_smalln_mma_kernel (small-batch warp-MMA)"}.get(kind0, "tc_q4_kernel")
        roof["per"] = "average over all launches of the step (every launch is this kernel family)"
    if tp_mode:
        roof["per"] += "; per GPU: each rank streams its own shards"
    res = {
        "metric": METRIC,
        "value": round(tok_s, 2),
        "unit": "tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 5),
        "higher_is_better": True,
        "scaling": "strong" if tp_mode else "weak",
        "vs_baseline": None,
        "dtype": "q4f16 (int4 codes x fp16 -> fp32 accumulate, fp16 out)",
        "data": "synthetic (seeded realistic q4f16 weights, N(0,1) fp16 x)",
        "config": {"workload": label,
                   "model": model, "tokens_per_step": n,
                   "layers_linears": len(mats), "weight_bytes": int(sum(inputs.q4_bytes(K, N) for _, K, N in mats)),
                   "parallelism": (f"megatron-tp{world}" if tp_mode else f"replicas{world}") if world > 1 else "single",
                   "l2": "not flushed: per-step working set %.2f GB >> 126 MB L2" % (bytes_step / 1e9),
                   "graph": graph is not None, "pdl": not args.no_pdl, "schedule": sched,
                   **({"tp_allreduce": tp_allreduce} if tp_mode else {})},
        "hbm_gbs": round(gbs, 1),
        "tflops": round(tflops, 3),
        "roofline": roof,
        "e2e": {"value": round(streams * n * args.steps / (ms_e2e / 1e3), 2), "unit": "tok/s",
                "h2d_bytes_per_step": int(x_host.numel() * 2), "d2h_bytes_per_step": int(out_host.numel() * 2),
                "how": "public API, captured step replayed; H2D of x and D2H of the logits inside the timed region"},
        "e2e_eager": {"value": round(streams * n * args.steps / (ms_eager / 1e3), 2), "unit": "tok/s",
                      "host_us_per_step": round(1e6 * host_eager_s / args.steps, 1),
                      "how": "every C-ABI call dispatched from Python each step (ctypes binding + host dispatch), "
                             "same copies"},
        "gpu_launches": launches * args.steps,
        "serial_chain": serial_line,
        "clocks": ck,
        "setup_s": round(t_gen, 1),
    }
    return res


def traffic_per_launch(workload, n):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(f"{workload}:n{n}")


# --------------------------------------------------------------------- oracle
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(workload, n, nthreads=None, which=None, budget_s=None):
    """Time the oracle (oracle.matmul_f64, full outputs) on a bounded sample of
    one step's workload.  which = i: only linear i of layer 0 (the reference arm
    rotates through them, one per step).  which = None: the layer set's linears
    in order until `budget_s` seconds of oracle time have run (default 10 s;
    for the 7B decode set on 16 cores that is the whole set, measured, not
    extrapolated).  Returns (tok/s, measured sample seconds, info): a partial
    sample is extrapolated by multiply-accumulate count,
    t_step = t_sample * MAC(set) / MAC(sample)."""
    import oracle
    model, mats = layer_set(workload)
    layer0 = [(nm, K, N) for nm, K, N in mats if nm.startswith("L0.")]
    sample = mats if which is None else [layer0[which % len(layer0)]]
    budget = 10.0 if budget_s is None else budget_s
    # all host cores the process may run on (torchrun sets OMP_NUM_THREADS=1)
    cores = nthreads or len(os.sched_getaffinity(0))
    gen = {}
    for nm, K, N in sample:
        if (K, N) not in gen:
            gen[(K, N)] = inputs.stress_weights(5 + K + N, K, N)
    xs = {K: inputs.activations(7 + n + K, n, K) for _, K, _ in sample}
    done = []
    t0 = time.perf_counter()
    for nm, K, N in sample:
        pk, sc = gen[(K, N)]
        oracle.matmul_f64(xs[K], pk, sc, K, N, nthreads=cores)
        done.append((nm, K, N))
        if which is None and time.perf_counter() - t0 > budget:
            break
    t_sample = time.perf_counter() - t0
    mac_sample = sum(n * K * N for _, K, N in done)
    mac_step = sum(n * K * N for _, K, N in mats)
    t_step = t_sample * mac_step / mac_sample
    if which is not None:
        what = "one linear of layer 0 per step (rotating q..down)"
    elif len(done) == len(mats):
        what = f"the whole {len(mats)}-linear layer set (measured, no extrapolation)"
    else:
        what = f"the first {len(done)} of the {len(mats)} linears of the layer set (a {budget:.0f} s budget)"
    tail = "" if len(done) == len(mats) else (f"; extrapolated by multiply-accumulate count to the "
                                              f"{len(mats)}-linear layer set")
    return n / t_step, t_sample, {"cores": cores,
                                  "sample": f"oracle (fp64, {cores} threads) on {what} at n={n}, full outputs{tail}"}


def run_reference(args):
    """The reference arm: the oracle, as it stands, on the host cores.  Each of
    the W warm-up and K timed steps times one bounded sample (one linear of
    layer 0, rotating); ms_per_step is the measured wall time of one sample
    (what the driver's clock sees), value the extrapolated whole-layer-set
    tok/s (median over the K steps)."""
    import oracle
    oracle.build()
    for i in range(args.warmup):
        oracle_sample(args.workload, args.n, which=i)
    vals, secs = [], []
    for i in range(args.steps):
        v, t, info = oracle_sample(args.workload, args.n, which=i)
        vals.append(v)
        secs.append(t)
    v = float(np.median(vals))
    # single-thread oracle on one sample (once)
    v1, t1, _ = oracle_sample(args.workload, args.n, nthreads=1, which=0)
    return {
        "metric": METRIC, "value": round(v, 6), "unit": "tok/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * float(np.median(secs)), 3),
        "ms_per_step_is": "measured wall time of one bounded oracle sample (value is extrapolated to the layer set)",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (oracle)", "data": "synthetic", "impl": "reference",
        "config": {"workload": args.workload, "tokens_per_step": args.n},
        "cpu_baseline": {"value": round(v, 6), "unit": "tok/s", "cores": info["cores"], "kind": "oracle",
                         "sample": info["sample"], "cpu_model": cpu_model(),
                         "single_thread": {"value": round(v1, 6), "unit": "tok/s", "sample_s": round(t1, 3)}},
        "e2e": {"value": round(v, 6), "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama2-7b-decode",
                    choices=["llama2-7b-decode", "llama2-13b-decode", "llama2-70b-decode",
                             "llama2-7b-prefill", "llama2-13b-prefill", "llama2-70b-prefill"])
    ap.add_argument("--n", type=int, default=None, help="tokens per step (decode: 1)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--tp-shard", type=int, default=1,
                    help="run rank 0's shard of a p-way tensor-parallel layer set on this GPU "
                         "(per-GPU compute-only time; no collective)")
    ap.add_argument("--serial", action="store_true",
                    help="every linear its own dependent call (default: q/k/v and gate/up, which read the same x, "
                         "as one relax_q4_matmul_grouped call each)")
    ap.add_argument("--fused", action="store_true",
                    help="stack q/k/v and gate/up rows into one call each (same weights)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="with N > 1 ranks: independent decode replicas instead of tensor parallelism")
    ap.add_argument("--tp", action="store_true",
                    help="tensor parallelism over the ranks even at N = 1 (one NCCL rank: exercises the "
                         "collectives of the TP step on one GPU); the default for N > 1")
    ap.add_argument("--chain", action="store_true",
                    help="n = 1: the whole layer set as one persistent launch (relax_q4_chain_run)")
    ap.add_argument("--nccl-allreduce", action="store_true",
                    help="TP decode: sum the row-parallel partials with an NCCL all_reduce instead of the fused "
                         "kernel epilogue (relax_q4_matmul_allreduce)")
    ap.add_argument("--kv", type=int, default=0,
                    help="with --block fused at n = 1: run the decode attention over a KV cache of this length "
                         "in every layer (relax_kv_append + relax_attn_decode), the whole decode step")
    ap.add_argument("--block", default="none", choices=["none", "fused", "unfused"],
                    help="decoder-block chain with RMSNorm / SiLU-mul / residual fused into the linears "
                         "(fused) or as separate kernels (unfused); implies the fused q/k/v, gate/up layout")
    args = ap.parse_args()
    if args.n is None:
        args.n = 1 if args.workload.endswith("decode") else 512
    if args.warmup < 3:
        args.warmup = 3
    if args.block != "none":
        args.fused = True

    under_torchrun = "WORLD_SIZE" in os.environ and "LOCAL_RANK" in os.environ
    if args.gpus > 1 and not under_torchrun:
        # one process per GPU: re-launch under torch.distributed.run (127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
               os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args)))
        return 0

    if world > 1 and not args.replicas:
        args.tp = True
    if world > 1 or args.tp:
        # NCCL logs to stdout (even its version line at NCCL_DEBUG=WARN): keep rank
        # 0's stdout the one JSON line by sending NCCL's log to stderr
        os.environ["NCCL_DEBUG"] = os.environ.get("RELAX_BENCH_NCCL_DEBUG", "WARN")
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if world == 1 and "MASTER_ADDR" not in os.environ:
            # a single self-launched rank picks its own port; a port taken
            # between the probe and the bind (EADDRINUSE) is retried with another
            for attempt in range(5):
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()), RANK="0", WORLD_SIZE="1")
                try:
                    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
                    break
                except dist.DistNetworkError:
                    if attempt == 4:
                        raise
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            v, t_s, info = oracle_sample(args.workload, args.n)
            v1, t1, info1 = oracle_sample(args.workload, args.n, nthreads=1, which=0)
            res["cpu_baseline"] = {"value": round(v, 6), "unit": "tok/s", "cores": info["cores"],
                                   "kind": "oracle", "sample": info["sample"], "sample_s": round(t_s, 3),
                                   "cpu_model": cpu_model(),
                                   "single_thread": {"value": round(v1, 6), "unit": "tok/s", "sample": info1["sample"],
                                                     "sample_s": round(t1, 3)}}
        print(json.dumps(res))
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
