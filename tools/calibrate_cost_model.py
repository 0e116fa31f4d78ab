"""Fit a B200 cost model for the overlap solver from measured timings
(reference fit_affine, overlap.cpp:36-63).

Samples, all in microseconds (the reference's cost units):
  ffa_fwd / ffa_bwd  (mask-aware pairs, us) of the FFA kernels at the CP
                     shape (48 q heads, 8 kv heads, head_dim 128), block-causal
                     masks of several sizes;
  cast / reduce      (tokens, us) of one NCCL all-to-all round carrying K+V
                     bf16 (4 KB / token) or dK+dV f32 (8 KB / token) plus the
                     gather / scatter-add kernels around it — only when run
                     under torchrun with >= 2 ranks.
Each set goes through the planner's own fit_affine (least squares, negative
coefficients clamped), and rank 0 writes configs/cost_model_b200.json.

    python tools/calibrate_cost_model.py                      # FFA terms only
    torchrun --nproc-per-node 2 tools/calibrate_cost_model.py  # + cast/reduce
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_13211_b200 import _lib  # noqa: E402
from paper_2505_13211_b200.ffa import FFAPlan, ffa_backward, ffa_forward  # noqa: E402
from paper_2505_13211_b200.planner import debug_eval  # noqa: E402

HQ, HK, D = 48, 8, 128


def _time_us(fn, iters=5) -> float:
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def ffa_samples(dev) -> tuple[list, list]:
    fwd, bwd = [], []
    for S, block in ((4096, 1024), (8192, 2048), (16384, 4096), (32768, 8192), (65536, 8192)):
        qr = [[i, i + block] for i in range(0, S, block)]
        kr = [[0, i + block] for i in range(0, S, block)]
        plan = FFAPlan(qr, kr, [0] * len(qr), S, S, D)
        area = plan.area()
        q = torch.randn(S, HQ, D, device=dev, dtype=torch.bfloat16)
        k = torch.randn(S, HK, D, device=dev, dtype=torch.bfloat16)
        v = torch.randn(S, HK, D, device=dev, dtype=torch.bfloat16)
        do = torch.randn(S, HQ, D, device=dev, dtype=torch.bfloat16)
        out, lse = ffa_forward(plan, q, k, v)
        fwd.append([int(area), int(round(_time_us(lambda: ffa_forward(plan, q, k, v, out=out, lse=lse))))])
        bwd.append([int(area), int(round(_time_us(lambda: ffa_backward(plan, q, k, v, out, lse, do))))])
        del q, k, v, do, out, lse
    return fwd, bwd


def comm_samples(dev, world: int) -> tuple[list, list]:
    import torch.distributed as dist

    cast, red = [], []
    for tokens in (2048, 8192, 32768, 131072):
        per_peer = tokens // world
        for bytes_per_token, acc in ((2 * HK * D * 2, cast), (2 * HK * D * 4, red)):
            n = per_peer * world * bytes_per_token // 4
            src = torch.randn(n, device=dev)
            dst = torch.empty_like(src)

            def step():
                dist.all_to_all_single(dst, src)
                if acc is red:
                    src.add_(dst)  # the scatter-add after the reduce exchange

            us = torch.tensor([_time_us(step)], device=dev)
            dist.all_reduce(us, op=dist.ReduceOp.MAX)
            acc.append([tokens, int(round(us.item()))])
    return cast, red


def main() -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.lib()
    model = {}
    fwd, bwd = ffa_samples(dev)
    for name, samples in (("ffa_fwd", fwd), ("ffa_bwd", bwd)):
        lat, per = debug_eval("fit_affine", samples=samples)
        model[name] = {"latency": lat, "per_unit": per, "samples": samples}
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        cast, red = comm_samples(dev, world)
        for name, samples in (("cast", cast), ("reduce", red)):
            lat, per = debug_eval("fit_affine", samples=samples)
            model[name] = {"latency": lat, "per_unit": per, "samples": samples}
        dist.destroy_process_group()
    if rank == 0:
        out = ROOT / "configs" / "cost_model_b200.json"
        out.parent.mkdir(exist_ok=True)
        prev = json.loads(out.read_text()) if out.exists() else {}
        prev.update(model)
        prev["_note"] = ("B200 timings (us) fitted with the planner's fit_affine; ffa_* per mask-aware pair at "
                         f"hq={HQ}, hk={HK}, d={D}; cast/reduce per token (tools/calibrate_cost_model.py)")
        out.write_text(json.dumps(prev, indent=1) + "\n")
        print(json.dumps({k: (v if k.startswith("_") else {kk: v[kk] for kk in ("latency", "per_unit")})
                          for k, v in prev.items()}, indent=1))


if __name__ == "__main__":
    main()
