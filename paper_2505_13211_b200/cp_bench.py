"""Multi-GPU leg of bench.py: context-parallel FFA fwd+bwd, weak scaling.

Workload: MAGI-1 24B attention shape (48 query
heads, 8 key/value heads, head_dim 128), block-causal with block 8192,
131072 tokens per rank (N=8 is the 1M-token sequence), greedy dispatch with
the default chunk (S/cp/8), GroupCast/GroupReduce over NCCL, stage count
from the overlap solver. `value` = whole-job mask-aware TFLOPS = total FLOPs
/ max-over-ranks device time.
"""
from __future__ import annotations

import json
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.distributed as dist

PER_RANK = 131072
HQ, HK, D, BLOCK = 48, 8, 128, 8192
# B200 cost model for the overlap solver: the fitted one when
# tools/calibrate_cost_model.py has been run (configs/cost_model_b200.json),
# else analytic figures (~800 TFLOPS FFA, ~300 GB/s effective cast).
COST = {"ffa_fwd": {"latency": 20, "per_unit": 4 * HQ * D / 8.0e8},
        "ffa_bwd": {"latency": 20, "per_unit": 10 * HQ * D / 6.0e8},
        "cast": {"latency": 30, "per_unit": (2 * HK * D * 2) / 3.0e5},
        "reduce": {"latency": 30, "per_unit": (2 * HK * D * 4) / 3.0e5}}
_FITTED = Path(__file__).resolve().parents[1] / "configs" / "cost_model_b200.json"
if _FITTED.exists():
    _fit = json.loads(_FITTED.read_text())
    COST.update({k: {"latency": v["latency"], "per_unit": v["per_unit"]} for k, v in _fit.items()
                 if k in COST and isinstance(v, dict)})


def scenario(cp: int) -> dict:
    S = PER_RANK * cp
    return {"workload": {"mask": {"seqlen": S, "pattern": "block_causal", "params": {"block_size": BLOCK}},
                         "num_heads_q": HQ, "num_heads_k": HK, "num_heads_v": HK, "head_dim": D},
            "cp_size": cp, "cost_model": COST,
            "overlap": {"min_chunk_size": 4096,
                        "max_num_chunks": int(os.environ.get("MAGI_CP_MAX_CHUNKS", "8"))}}


def config(world: int, mode: str = "magi") -> dict:
    """The N>1 line's `config` (shared with the reference arm), computed on
    the host from the planner alone."""
    S = PER_RANK * world
    if mode == "ring":
        chunk, ns = S // (2 * world), (world, world)
    elif mode == "ulysses":
        chunk, ns = S // world, (1, 1)
    else:
        from .planner import Scenario

        xp = Scenario(scenario(world)).exec_plan()
        chunk, ns = xp["chunk_size"], (xp["num_stages_fwd"], xp["num_stages_bwd"])
    area = block_causal_area(S, BLOCK)
    fwd = 4 * area * HQ * D
    return {"workload": "cp_block_causal_magi1_24b", "seqlen": S, "tokens_per_rank": PER_RANK,
            "num_heads_q": HQ, "num_heads_k": HK, "head_dim": D, "mask": f"block_causal(block={BLOCK})",
            "area_multiplicity": area, "flops_per_step": fwd + fwd * 5 // 2,
            "dispatch": {"ring": "zigzag", "ulysses": "contiguous"}.get(mode, "greedy"), "cp_mode": mode,
            "dispatch_chunk_size": chunk, "num_stages_fwd": ns[0], "num_stages_bwd": ns[1],
            "parallelism": f"cp{world}", "l2": "inputs larger than L2 per rank; no flush"}


def block_causal_area(S: int, block: int) -> int:
    n = S // block
    return n * (n + 1) // 2 * block * block


def anchor(steps: int = 2, warmup: int = 1) -> dict:
    """The weak-scaling anchor: the N>1 workload's per-rank shape at cp = 1
    (131072 tokens, 48 q / 8 kv heads, block-causal 8192) through the same
    CPAttention executor on one GPU (host-local FFA only). Weak efficiency at
    N is tflops_per_gpu(N) / this value."""
    from .cp import CPAttention

    dev = torch.device("cuda", torch.cuda.current_device())
    cpa = CPAttention(scenario(1), HQ, HK, D)
    L = cpa.local_tokens
    g = torch.Generator(device="cpu").manual_seed(1234)
    q = torch.randn(L, HQ, D, generator=g).to(torch.bfloat16).to(dev)
    k = torch.randn(L, HK, D, generator=g).to(torch.bfloat16).to(dev)
    v = torch.randn(L, HK, D, generator=g).to(torch.bfloat16).to(dev)
    do = torch.randn(L, HQ, D, generator=g).to(torch.bfloat16).to(dev)

    def step():
        out, lse, out32 = cpa.forward(q, k, v)
        return cpa.backward(q, k, v, out32, lse, do)

    for _ in range(warmup):
        step()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    fwd, bwd = cpa.flops()
    return {"what": "CP workload per-rank shape at cp=1 (weak-scaling anchor)", "config": config(1),
            "steps": steps, "warmup": warmup, "ms_per_step": ms,
            "tflops_per_gpu": (fwd + bwd) / (ms * 1e-3) / 1e12}


def run(args) -> None:
    from bench import METRIC, UNIT, ClockSampler, _peaks
    from paper_2505_13211_b200.cp import CPAttention

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the bench's stdout is one JSON line: native libraries (NCCL prints its
    # version banner at communicator init) write to fd 1 only as stderr; the
    # JSON line goes to the saved stdout descriptor
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    dist.init_process_group("nccl", device_id=dev)
    mode = getattr(args, "cp_mode", "magi")
    ring = mode == "ring"
    uly = mode == "ulysses"
    if ring:
        from paper_2505_13211_b200.ring import RingAttention

        cpa = RingAttention(scenario(world)["workload"]["mask"], HQ, HK, D)
    elif uly:
        from paper_2505_13211_b200.ulysses import UlyssesAttention

        cpa = UlyssesAttention(scenario(world)["workload"]["mask"], HQ, HK, D)
    elif mode in ("capi", "capi_p2p"):
        from paper_2505_13211_b200.cp import CPExecutorC

        cpa = CPExecutorC(scenario(world), HQ, HK, D, transport="p2p" if mode == "capi_p2p" else "nccl")
    else:
        cpa = CPAttention(scenario(world), HQ, HK, D, transport="p2p" if mode == "p2p" else "nccl")
    L = cpa.local_tokens
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    q_h = torch.randn(L, HQ, D, generator=g).to(torch.bfloat16).pin_memory()
    k_h = torch.randn(L, HK, D, generator=g).to(torch.bfloat16).pin_memory()
    v_h = torch.randn(L, HK, D, generator=g).to(torch.bfloat16).pin_memory()
    do_h = torch.randn(L, HQ, D, generator=g).to(torch.bfloat16).pin_memory()
    q, k, v, do = (t.to(dev) for t in (q_h, k_h, v_h, do_h))

    def step():
        out, lse, out32 = cpa.forward(q, k, v)
        return cpa.backward(q, k, v, out32, lse, do)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)

    # e2e: host buffers in, gradients out, every step
    o_h = torch.empty(L, HQ, D, dtype=torch.bfloat16).pin_memory()
    dq_h = torch.empty(L, HQ, D, dtype=torch.bfloat16).pin_memory()
    dk_h = torch.empty(L, HK, D, dtype=torch.bfloat16).pin_memory()
    dv_h = torch.empty(L, HK, D, dtype=torch.bfloat16).pin_memory()

    # two device input sets: step i+1's inputs travel (H2D stream) and step
    # i-1's gradients return (D2H stream) while step i computes; every step
    # still copies its own inputs in and its gradients out
    sets = [dict(q=q, k=k, v=v, do=do), {n: torch.empty_like(t) for n, t in dict(q=q, k=k, v=v, do=do).items()}]
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def e2e_run(n, start=None):
        mk = lambda: [torch.cuda.Event() for _ in range(n)]  # noqa: E731
        ev_qkv, ev_do, ev_done, ev_out = mk(), mk(), mk(), mk()
        keep = []

        def h2d(i):
            b = sets[i % 2]
            with torch.cuda.stream(h2d_s):
                if i == 0 and start is not None:
                    h2d_s.wait_event(start)
                if i >= 2:
                    h2d_s.wait_event(ev_done[i - 2])  # step i-2 finished reading this set
                for name, src in (("q", q_h), ("k", k_h), ("v", v_h)):
                    b[name].copy_(src, non_blocking=True)
                ev_qkv[i].record(h2d_s)
                b["do"].copy_(do_h, non_blocking=True)
                ev_do[i].record(h2d_s)

        h2d(0)
        for i in range(n):
            if i + 1 < n:
                h2d(i + 1)
            b = sets[i % 2]
            stream.wait_event(ev_qkv[i])
            out, lse, out32 = cpa.forward(b["q"], b["k"], b["v"])
            ev_fwd = torch.cuda.Event()
            ev_fwd.record(stream)
            with torch.cuda.stream(d2h_s):  # O travels back while the backward computes
                d2h_s.wait_event(ev_fwd)
                o_h.copy_(out, non_blocking=True)
                out.record_stream(d2h_s)
            stream.wait_event(ev_do[i])
            grads = cpa.backward(b["q"], b["k"], b["v"], out32, lse, b["do"])
            ev_done[i].record(stream)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_done[i])
                for dst, g in zip((dq_h, dk_h, dv_h), grads):
                    dst.copy_(g, non_blocking=True)
                    g.record_stream(d2h_s)
                ev_out[i].record(d2h_s)
            keep.append(grads)
        stream.wait_event(ev_out[n - 1])

    e2e_steps = max(1, min(args.steps, 3))
    e2e_run(1)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    e2e_run(e2e_steps, start=e0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / e2e_steps], device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    clk = clocks.stop() if rank == 0 else None

    fwd, bwd = cpa.flops()
    total = fwd + bwd
    comm_keys = list(cpa.comm_tokens().keys())
    comm = torch.tensor([list(cpa.comm_tokens().values()) or [0.0]], dtype=torch.float64, device=dev)
    dist.all_reduce(comm)
    if rank == 0:
        cfg = config(world, mode)
        assert cfg["flops_per_step"] == total, (cfg["flops_per_step"], total)
        peaks = _peaks()
        value = total / (ms.item() * 1e-3) / 1e12
        per_gpu = value / world
        n_launch = 0
        if uly:
            n_launch = 1 + 1 + 1 + 3  # fwd, cast, preprocess, dkdv + dq + final casts inside ffa_bwd
        elif ring:
            n_plans = sum(p is not None for p in cpa.plans)
            n_launch = n_plans * 3 + 1 + 1 + 3  # fwd + dq + dkdv per plan, cast, preprocess, final casts
        elif mode == "capi":
            nf, nb = cpa.xplan["num_stages_fwd"], cpa.xplan["num_stages_bwd"]
            # host fwd + per stage (gather x2, ffa), cast; preprocess, host bwd (2), per stage
            # (gather x2, dkdv, dq, scatter-adds), final casts
            n_launch = 2 + 3 * nf + 1 + 3 + 4 * nb + 2 * world * nb + 3
        elif mode == "capi_p2p":
            nf, nb = cpa.xplan["num_stages_fwd"], cpa.xplan["num_stages_bwd"]
            # fwd per stage: cast (wait, 2 copies, signal), wait, ffa, signal; bwd per stage: cast,
            # 2 waits, dkdv + dq, 2 signals, reduce (wait, 2 scatter-adds per consumer, signal)
            # (+ the end-of-pass wait on the owners' reads), final casts
            n_launch = 2 + 7 * nf + 1 + 3 + (4 + 6 + 2 + 2 * (world - 1) + 1) * nb + 3
        else:
            for st in cpa.fwd_stages:
                # p2p: flag wait + 2 copies + signal on the comm stream, wait + signal beside the FFA
                n_launch += 1 + (6 if mode == "p2p" else 2 * (1 if sum(st.send_splits) else 0))
            if mode == "p2p":
                # per stage: cast (wait, 2 copies, signal), compute (2 waits, dK/dV + dQ, 2 signals),
                # reduce (wait, 2 scatter-adds per consumer, signal)
                for P in cpa._p2p_bwd:  # (+ the end-of-pass wait on the owners' reads)
                    n_launch += 4 + 6 + 2 + 2 * len(P["per_dst"]) + 1
            else:
                for st in cpa.bwd_stages:
                    n_launch += 2 + 2 * (1 if sum(st.send_splits) else 0) + 2 * world
            n_launch += 2 + 1 + 2 + 3  # host fwd + cast, preprocess, host bwd (2), final casts
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms.item(), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": cfg,
            "tokens_per_s": PER_RANK * world / (ms.item() * 1e-3),
            "comm_tokens_all_ranks": dict(zip(comm_keys, comm[0].tolist())),
            "roofline": {"bound": "tensor", "kernel": "whole CP step", "achieved": per_gpu,
                         "peak": peaks["bf16"], "unit": "TFLOP/s", "frac": per_gpu / peaks["bf16"],
                         "traffic": None, "peak_source": peaks["source"]},
            "tflops_per_gpu": per_gpu,
            "e2e": {"value": total / (e2e_ms.item() * 1e-3) / 1e12, "unit": UNIT,
                    "h2d_bytes_per_step": sum(t.numel() * 2 for t in (q_h, k_h, v_h, do_h)),
                    "d2h_bytes_per_step": sum(t.numel() * 2 for t in (o_h, dq_h, dk_h, dv_h)),
                    "copies": "H2D q, k, v, dO; D2H O, dQ, dK, dV (bf16), every step",
                    "ms_per_step": e2e_ms.item(), "per_rank": True},
            "clocks": clk,
            "gpu_launches": n_launch * args.steps,
        }
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    dist.barrier()
    dist.destroy_process_group()
