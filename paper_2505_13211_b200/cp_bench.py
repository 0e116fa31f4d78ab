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
    else:
        cpa = CPAttention(scenario(world), HQ, HK, D)
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
    comm = torch.tensor([list(cpa.comm_tokens().values())], dtype=torch.float64, device=dev)
    dist.all_reduce(comm)
    if rank == 0:
        peaks = _peaks()
        value = total / (ms.item() * 1e-3) / 1e12
        per_gpu = value / world
        n_launch = 0
        if uly:
            n_launch = 1 + 1 + 1 + 3  # fwd, cast, preprocess, dkdv + dq + final casts inside ffa_bwd
        elif ring:
            n_plans = sum(p is not None for p in cpa.plans)
            n_launch = n_plans * 3 + 1 + 1 + 3  # fwd + dq + dkdv per plan, cast, preprocess, final casts
        else:
            for st in cpa.fwd_stages:
                n_launch += 1 + 2 * (1 if sum(st.send_splits) else 0)
            for st in cpa.bwd_stages:
                n_launch += 2 + 2 * (1 if sum(st.send_splits) else 0) + 2 * world
            n_launch += 2 + 1 + 2 + 3  # host fwd + cast, preprocess, host bwd (2), final casts
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms.item(), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "cp_block_causal_magi1_24b", "seqlen": PER_RANK * world,
                       "tokens_per_rank": PER_RANK, "num_heads_q": HQ, "num_heads_k": HK, "head_dim": D,
                       "mask": f"block_causal(block={BLOCK})", "dispatch": "zigzag" if ring else ("contiguous" if uly else "greedy"),
                       "cp_mode": mode,
                       "dispatch_chunk_size": cpa.local_tokens if uly else cpa.chunk_size,
                       "num_stages_fwd": world if ring else (1 if uly else cpa.xplan["num_stages_fwd"]),
                       "num_stages_bwd": world if ring else (1 if uly else cpa.xplan["num_stages_bwd"]),
                       "parallelism": f"cp{world}",
                       "flops_per_step": total,
                       "tokens_per_s": PER_RANK * world / (ms.item() * 1e-3),
                       "comm_tokens_all_ranks": dict(zip(cpa.comm_tokens().keys(), comm[0].tolist())),
                       "l2": "inputs larger than L2 per rank; no flush"},
            "roofline": {"bound": "tensor", "kernel": "whole CP step", "achieved": per_gpu,
                         "peak": peaks["bf16"], "unit": "TFLOP/s", "frac": per_gpu / peaks["bf16"],
                         "traffic": None, "peak_source": peaks["source"]},
            "tflops_per_gpu": per_gpu,
            "e2e": {"value": total / (e2e_ms.item() * 1e-3) / 1e12, "unit": UNIT,
                    "h2d_bytes_per_step": sum(t.numel() * 2 for t in (q_h, k_h, v_h, do_h)),
                    "d2h_bytes_per_step": sum(t.numel() * 2 for t in (dq_h, dk_h, dv_h)),
                    "ms_per_step": e2e_ms.item(), "per_rank": True},
            "clocks": clk,
            "gpu_launches": n_launch * args.steps,
        }
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    dist.barrier()
    dist.destroy_process_group()
