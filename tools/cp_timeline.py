"""Per-stage CUDA-event timeline of the context-parallel step (cp.py) and the
stage-pipeline estimate it should match (reference sim.cpp:193-248).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/cp_timeline.py --per-rank 32768 --stages 4 --out profiles/cp_timeline.json

Every rank runs forward + backward of a block-causal scenario whose stage
count is forced (a cost model under which splitting is free, `max_num_chunks`
packages), with CUDA events around each task on its own stream:
    fwd step j:  cast(j+1) on the comm stream || ffa(j) on the compute stream
    bwd step j:  cast(j+1) || ffa(j) || reduce(j-1) on the reduce stream,
                 then the final reduce exposed.
Rank 0 writes the spans of every rank (ms from the pass start), the measured
overlaps (cast(j+1) ∩ ffa(j), reduce(j) ∩ ffa(j+1)), the exposed tail after
the last FFA, and the reference's stage-pipeline estimate evaluated on the
same stage plan with the fitted B200 cost model (configs/cost_model_b200.json)
next to the measured pass time.
"""
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

STAGED = {"ffa_fwd": {"latency": 0, "per_unit": 8.19e-05}, "ffa_bwd": {"latency": 0, "per_unit": 2.05e-04},
          "cast": {"latency": 0, "per_unit": 0.082}, "reduce": {"latency": 0, "per_unit": 0.082}}


def affine(c: dict, work: int) -> float:
    return 0.0 if work <= 0 else max(0.0, c["latency"] + c["per_unit"] * work)


def estimate(host_pairs, stage_pairs, stage_tokens, cm, backward: bool) -> float:
    """Stage pipeline of simulate_magi (sim.cpp:193-248), in µs: step j
    starts when every task of step j-1 has finished."""
    ffa = cm["ffa_bwd" if backward else "ffa_fwd"]
    s = len(stage_pairs)
    total = 0.0
    for j in range(s + 1):
        step = [affine(ffa, host_pairs if j == 0 else stage_pairs[j - 1])]
        if j + 1 <= s:
            step.append(affine(cm["cast"], stage_tokens[j]))
        if backward and j >= 2:
            step.append(affine(cm["reduce"], stage_tokens[j - 2]))
        total += max(step)
    if backward and s:
        total += affine(cm["reduce"], stage_tokens[s - 1])
    return total


def overlap(a, b) -> float:
    return max(0.0, min(a["end_ms"], b["end_ms"]) - max(a["start_ms"], b["start_ms"]))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-rank", type=int, default=32768)
    ap.add_argument("--block", type=int, default=4096)
    ap.add_argument("--stages", type=int, default=4)
    ap.add_argument("--hq", type=int, default=48)
    ap.add_argument("--hk", type=int, default=8)
    ap.add_argument("--out", default="")
    ap.add_argument("--bench", action="store_true",
                    help="the bench's own scenario (cp_bench.scenario: fitted B200 cost model, solver's stages)")
    args = ap.parse_args()

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2505_13211_b200.cp import CPAttention

    S, D = args.per_rank * world, 128
    scen = {"workload": {"mask": {"seqlen": S, "pattern": "block_causal", "params": {"block_size": args.block}},
                         "num_heads_q": args.hq, "num_heads_k": args.hk, "num_heads_v": args.hk, "head_dim": D},
            "cp_size": world, "cost_model": STAGED,
            "overlap": {"min_chunk_size": 512, "max_num_chunks": args.stages}}
    if args.bench:
        from paper_2505_13211_b200 import cp_bench

        scen = cp_bench.scenario(world)
        args.per_rank, args.block, args.hq, args.hk = cp_bench.PER_RANK, cp_bench.BLOCK, cp_bench.HQ, cp_bench.HK
        S = args.per_rank * world
        args.stages = None
    cpa = CPAttention(scen, args.hq, args.hk, D)
    L = cpa.local_tokens
    g = torch.Generator(device="cpu").manual_seed(rank)
    q = torch.randn(L, args.hq, D, generator=g).to(torch.bfloat16).to(dev)
    k = torch.randn(L, args.hk, D, generator=g).to(torch.bfloat16).to(dev)
    v = torch.randn(L, args.hk, D, generator=g).to(torch.bfloat16).to(dev)
    do = torch.randn(L, args.hq, D, generator=g).to(torch.bfloat16).to(dev)
    for _ in range(2):
        o, lse, o32 = cpa.forward(q, k, v)
        cpa.backward(q, k, v, o32, lse, do)
    torch.cuda.synchronize()
    dist.barrier()
    stream = torch.cuda.current_stream(dev)
    cpa.timeline = []
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t2 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    o, lse, o32 = cpa.forward(q, k, v)
    t1.record(stream)
    cpa.backward(q, k, v, o32, lse, do)
    t2.record(stream)
    torch.cuda.synchronize()
    spans = cpa.timeline_ms(t0)
    bwd_origin = t0.elapsed_time(t1)
    for sp in spans:  # backward spans relative to the backward's start
        if sp["pass"] == "bwd":
            sp["start_ms"] -= bwd_origin
            sp["end_ms"] -= bwd_origin
    pass_ms = {"fwd": t0.elapsed_time(t1), "bwd": t1.elapsed_time(t2)}

    cm = json.loads((ROOT / "configs" / "cost_model_b200.json").read_text())
    hp = cpa.host_plan.area() if cpa.host_plan is not None else 0
    est = {}
    for key, stages, bwd in (("fwd", cpa.fwd_stages, False), ("bwd", cpa.bwd_stages, True)):
        pairs = [st.plan.area() if st.plan is not None else 0 for st in stages]
        toks = [st.buf_tokens for st in stages]
        est[key] = {"estimate_ms": estimate(hp, pairs, toks, cm, bwd) / 1e3, "stage_pairs": pairs,
                    "stage_tokens": toks, "host_pairs": hp}

    def by(pass_, task):
        return {sp["stage"]: sp for sp in spans if sp["pass"] == pass_ and sp["task"] == task}

    fc, ff = by("fwd", "cast"), by("fwd", "ffa")
    bc, bf, br = by("bwd", "cast"), by("bwd", "ffa"), by("bwd", "reduce")
    last_ffa = max(bf) if bf else 0
    # the executor issues every GroupCast as soon as the comm stream is free
    # (all of them typically land during ffa(0)), so a cast is hidden when
    # it ends before the FFA step that consumes it could start; what is left
    # exposed is the wait of ffa(j) past the end of ffa(j-1)
    summary = {
        "fwd_cast_overlap_ms": {f"cast({j})": overlap(fc[j], ff[0]) for j in fc},
        "fwd_cast_exposed_ms": {f"cast({j})": max(0.0, fc[j]["end_ms"] - ff[j - 1]["end_ms"]) for j in fc},
        "bwd_cast_exposed_ms": {f"cast({j})": max(0.0, bc[j]["end_ms"] - bf[j - 1]["end_ms"]) for j in bc},
        "bwd_reduce_overlap_ms": {f"reduce({j})|ffa({j + 1})": overlap(br[j], bf[j + 1]) for j in br if j + 1 in bf},
        "bwd_exposed_tail_ms": max(0.0, max((s_["end_ms"] for s_ in br.values()), default=0.0)
                                   - bf[last_ffa]["end_ms"]) if bf else 0.0,
        "fwd_compute_ms": sum(x["end_ms"] - x["start_ms"] for x in ff.values()),
        "bwd_compute_ms": sum(x["end_ms"] - x["start_ms"] for x in bf.values()),
    }
    rec = {"rank": rank, "num_stages_fwd": cpa.xplan["num_stages_fwd"],
           "num_stages_bwd": cpa.xplan["num_stages_bwd"], "pass_ms": pass_ms, "estimate": est,
           "summary": summary, "spans": spans}
    allrec = [None] * world
    dist.all_gather_object(allrec, rec)
    if rank == 0:
        report = {"what": "cp.py per-stage CUDA-event timeline vs the stage-pipeline estimate",
                  "config": {"world": world, "per_rank_tokens": args.per_rank, "seqlen": S,
                             "mask": f"block_causal({args.block})", "hq": args.hq, "hk": args.hk, "d": D,
                             "forced_packages": args.stages},
                  "gpu": torch.cuda.get_device_name(dev), "ranks": allrec}
        text = json.dumps(report, indent=1)
        if args.out:
            Path(args.out).write_text(text)
        for r in allrec:
            print(json.dumps({k_: r[k_] for k_ in ("rank", "num_stages_fwd", "num_stages_bwd", "pass_ms")}
                             | {"est_ms": {p: r["estimate"][p]["estimate_ms"] for p in ("fwd", "bwd")}}
                             | r["summary"]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
