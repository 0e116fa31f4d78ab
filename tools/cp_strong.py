"""Strong scaling of the context-parallel step (SURVEY §8d config 5, strong
leg): a fixed sequence (default 1,048,576 tokens, block-causal 8192, 48 q /
8 kv heads, d = 128) split over N ranks, fwd + bwd through CPAttention with
the bench's scenario settings (greedy dispatch, default chunk S/cp/8, fitted
B200 cost model).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/cp_strong.py [--seqlen 1048576] [--steps 1] [--warmup 1]

Rank 0 prints one JSON line: ms per step (max over ranks, CUDA events) and
TFLOPS per GPU = FLOPs / (t * N) (Eq. 15, reference sim.cpp:36-45)."""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqlen", type=int, default=1048576)
    ap.add_argument("--block", type=int, default=8192)
    ap.add_argument("--hq", type=int, default=48)
    ap.add_argument("--hk", type=int, default=8)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2505_13211_b200 import cp_bench
    from paper_2505_13211_b200.cp import CPAttention

    D = 128
    scen = {"workload": {"mask": {"seqlen": args.seqlen, "pattern": "block_causal",
                                  "params": {"block_size": args.block}},
                         "num_heads_q": args.hq, "num_heads_k": args.hk, "num_heads_v": args.hk, "head_dim": D},
            "cp_size": world, "cost_model": cp_bench.COST,
            "overlap": {"min_chunk_size": 4096, "max_num_chunks": 8}}
    cpa = CPAttention(scen, args.hq, args.hk, D)
    L = cpa.local_tokens
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    q = torch.randn(L, args.hq, D, generator=g).to(torch.bfloat16).to(dev)
    k = torch.randn(L, args.hk, D, generator=g).to(torch.bfloat16).to(dev)
    v = torch.randn(L, args.hk, D, generator=g).to(torch.bfloat16).to(dev)
    do = torch.randn(L, args.hq, D, generator=g).to(torch.bfloat16).to(dev)

    def step():
        out, lse, out32 = cpa.forward(q, k, v)
        return cpa.backward(q, k, v, out32, lse, do)

    for _ in range(args.warmup):
        step()
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
    S, b = args.seqlen, args.block
    n = S // b
    area = n * (n + 1) // 2 * b * b
    fwd = 4 * area * args.hq * D
    flops = fwd + fwd * 5 // 2
    if rank == 0:
        print(json.dumps({"what": "CP strong scaling (fixed sequence)", "n_gpus": world, "seqlen": S,
                          "tokens_per_rank": L, "block": b, "hq": args.hq, "hk": args.hk, "head_dim": D,
                          "num_stages_fwd": cpa.xplan["num_stages_fwd"],
                          "num_stages_bwd": cpa.xplan["num_stages_bwd"], "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms.item(),
                          "tflops_per_gpu": flops / (ms.item() * 1e-3) / 1e12 / world,
                          "gpu": torch.cuda.get_device_name(dev)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
