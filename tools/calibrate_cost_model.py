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
coefficients clamped); the FFA latency terms are raised to the measured
per-stage overhead (the same per-rank mask as one call vs split by key
columns, stage_overhead_us), because a single call's intercept is ~0 while
splitting the work into stages is not free. Rank 0 writes
configs/cost_model_b200.json.

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


def stage_overhead_us(dev, S: int = 131072, block: int = 8192, pieces: int = 4) -> tuple[float, float]:
    """Per-stage fixed cost of the FFA at the CP per-rank size: the same mask
    run as one call vs split into `pieces` key-column ranges (the way stages
    split the remote K/V), each piece merged with the fused LSE-merge /
    accumulate epilogue. Returns (fwd, bwd) extra microseconds per piece."""
    from paper_2505_13211_b200.planner import debug_eval

    mask = {"seqlen": S, "pattern": "block_causal", "params": {"block_size": block}}
    cs = S // pieces

    def plan_of(col_chunks):
        sl = debug_eval("chunk_pair_slices", mask=mask, chunk=cs, q_chunks=list(range(pieces)),
                        k_chunks=col_chunks)
        return FFAPlan([x[0:2] for x in sl], [x[2:4] for x in sl], [x[4] for x in sl], S,
                       len(col_chunks) * cs, D) if sl else None

    whole = plan_of(list(range(pieces)))
    q = torch.randn(S, HQ, D, device=dev, dtype=torch.bfloat16)
    k = torch.randn(S, HK, D, device=dev, dtype=torch.bfloat16)
    v = torch.randn(S, HK, D, device=dev, dtype=torch.bfloat16)
    do = torch.randn(S, HQ, D, device=dev, dtype=torch.bfloat16)
    out = torch.zeros(S, HQ, D, device=dev, dtype=torch.float32)
    lse = torch.full((HQ, S), float("-inf"), device=dev)
    ks = [k[c * cs:(c + 1) * cs] for c in range(pieces)]
    vs = [v[c * cs:(c + 1) * cs] for c in range(pieces)]
    pk = [(pl, ks[c], vs[c]) for c, pl in enumerate(plan_of([c]) for c in range(pieces)) if pl is not None]

    def fwd_whole():
        ffa_forward(whole, q, k, v, out=out, lse=lse, accumulate=True)

    def fwd_parts():
        for pl, kk, vv in pk:
            ffa_forward(pl, q, kk, vv, out=out, lse=lse, accumulate=True)

    t1, tn = _time_us(fwd_whole, 2), _time_us(fwd_parts, 2)
    o_bf, lse2 = ffa_forward(whole, q, k, v)
    dq = torch.zeros(S, HQ, D, device=dev, dtype=torch.float32)
    dk = torch.zeros(S, HK, D, device=dev, dtype=torch.float32)
    dv = torch.zeros_like(dk)

    # as the CP executor runs a stage: delta once per pass, then dQ (accumulate)
    # and a fresh f32 dK/dV partial per stage
    L = _lib.lib()
    sp = torch.cuda.current_stream(dev).cuda_stream
    delta = torch.empty((HQ, S), dtype=torch.float32, device=dev)
    _lib.check(L.magiplan_ffa_bwd_preprocess(o_bf.data_ptr(), do.data_ptr(), delta.data_ptr(), S, HQ, D,
                                             _lib.BF16, sp))
    scale = D ** -0.5

    def bwd_calls(pl, kk, vv, dkk, dvv):
        _lib.check(L.magiplan_ffa_bwd_stage(pl.handle, q.data_ptr(), kk.data_ptr(), vv.data_ptr(), lse2.data_ptr(),
                                            delta.data_ptr(), do.data_ptr(), dq.data_ptr(), dkk.data_ptr(),
                                            dvv.data_ptr(), HQ, HK, scale, sp))

    def bwd_whole():
        bwd_calls(whole, k, v, dk, dv)

    def bwd_parts():
        for c, (pl, kk, vv) in enumerate(pk):
            bwd_calls(pl, kk, vv, dk[c * cs:(c + 1) * cs], dv[c * cs:(c + 1) * cs])

    b1, bn = _time_us(bwd_whole, 2), _time_us(bwd_parts, 2)
    n = len(pk)
    return max(0.0, (tn - t1) / max(n - 1, 1)), max(0.0, (bn - b1) / max(n - 1, 1))


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
    # the fitted intercept of a single call is ~0; what a stage really costs on
    # top of its pairs is the split overhead, measured at the CP per-rank size
    over_f, over_b = stage_overhead_us(dev)
    for name, samples, over in (("ffa_fwd", fwd, over_f), ("ffa_bwd", bwd, over_b)):
        lat, per = debug_eval("fit_affine", samples=samples)
        model[name] = {"latency": max(lat, over), "per_unit": per, "samples": samples,
                       "stage_overhead_us": over}
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
