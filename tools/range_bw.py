"""Roofline of the CP data-movement kernels: Range Gather of
K/V rows (bf16) and the deterministic Range Scatter-Reduce of dK/dV partials
(f32), at the bench's cp=8 shape, against the measured HBM copy bandwidth.

    python tools/range_bw.py [--json out.json]

Ranges are the real GroupCast send lists of the 1M-token cp8 bench scenario
(rank 0's stage-1 sends: `magiplan_scenario_exec_plan`), one K head group
(8 kv heads x 128 x 2 B = 2 KB per token row). Algorithmic bytes: gather
reads + writes every row once (2 x rows x row_bytes); scatter-add reads the
packed partial and read-modify-writes the destination (3 x rows x
row_bytes; one call per peer as in the GroupReduce, so a destination row
is read-modified-written once per peer and repeat visits can hit L2, which
is why the algorithmic rate may exceed the copy peak). Times: CUDA events
around 20 back-to-back repetitions after warm-up.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2505_13211_b200 import _lib, cp_bench  # noqa: E402
from paper_2505_13211_b200.cp import _stage_layouts  # noqa: E402
from paper_2505_13211_b200.planner import Scenario  # noqa: E402


def timed(fn, n=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    xp = Scenario(cp_bench.scenario(8)).exec_plan()
    L = xp["local_tokens"]
    # the largest send list of any rank's stage 1 (what one GroupCast gathers)
    best = None
    for r in range(8):
        for st in _stage_layouts(xp, r, "fwd_stages"):
            if best is None or sum(st.send_splits) > sum(best.send_splits):
                best = st
    ranges = best.send_ranges
    rows = sum(b - a for a, b in ranges)
    HK, D = cp_bench.HK, cp_bench.D
    r_t = torch.tensor(ranges, dtype=torch.int64, device=dev).reshape(-1, 2)
    offs, acc = [], 0
    for a, b in ranges:
        offs.append(acc)
        acc += b - a
    o_t = torch.tensor(offs, dtype=torch.int64, device=dev)
    Lib = _lib.lib()
    stream = torch.cuda.current_stream(dev).cuda_stream
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]

    src = torch.randn(L, HK, D, device=dev).to(torch.bfloat16)
    dst = torch.empty(rows, HK, D, device=dev, dtype=torch.bfloat16)
    rb = HK * D * 2
    g_ms = timed(lambda: _lib.check(Lib.magiplan_range_gather(src.data_ptr(), dst.data_ptr(), r_t.data_ptr(),
                                                              o_t.data_ptr(), len(ranges), rows, rb, stream)))
    g_bytes = 2 * rows * rb
    # correctness spot check
    ref = torch.cat([src[a:b] for a, b in ranges])
    assert torch.equal(ref, dst)

    # scatter-add as the GroupReduce runs it: one call per peer (its ranges
    # never alias within a call), peers in rank order
    part = torch.randn(rows, HK, D, device=dev)
    acc32 = torch.zeros(L, HK, D, device=dev)
    calls = []
    for dst_rank, idx in enumerate(best.send_by_dst):
        if not idx:
            continue
        rr = [ranges[i] for i in idx]
        o0 = offs[idx[0]]
        po, acc_ = [], 0
        for a, b in rr:
            po.append(acc_)
            acc_ += b - a
        calls.append((torch.tensor(rr, dtype=torch.int64, device=dev).reshape(-1, 2),
                      torch.tensor(po, dtype=torch.int64, device=dev), len(rr), acc_, o0))

    def scatter_all():
        for rt, ot, nr, nrows, o0 in calls:
            _lib.check(Lib.magiplan_range_scatter_add_f32(part[o0:].data_ptr(), acc32.data_ptr(), rt.data_ptr(),
                                                          ot.data_ptr(), nr, nrows, HK * D, stream))

    s_ms = timed(scatter_all)
    s_bytes = 3 * rows * HK * D * 4
    # correctness: one pass from zero against torch
    acc32.zero_()
    scatter_all()
    ref32 = torch.zeros_like(acc32)
    pos = 0
    for a, b in ranges:
        ref32[a:b] += part[pos:pos + (b - a)]
        pos += b - a
    torch.cuda.synchronize()
    assert torch.allclose(acc32, ref32, atol=1e-5, rtol=1e-5)
    copy_ms = timed(lambda: dst.copy_(ref))
    res = {"what": "Range Gather / Scatter-Reduce roofline (HBM-bound byte movement)",
           "scenario": "1M-token block-causal cp8 bench scenario, largest stage-1 send list",
           "num_ranges": len(ranges), "rows": rows, "row_bytes_gather": rb, "row_bytes_scatter": HK * D * 4,
           "gather": {"ms": g_ms, "bytes": g_bytes, "gbs": g_bytes / g_ms / 1e6, "frac": g_bytes / g_ms / 1e6 / peak},
           "scatter_add_f32": {"calls": len(calls), "ms": s_ms, "bytes": s_bytes, "gbs": s_bytes / s_ms / 1e6,
                               "frac": s_bytes / s_ms / 1e6 / peak},
           "torch_copy_same_bytes": {"ms": copy_ms, "gbs": g_bytes / copy_ms / 1e6},
           "peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
           "gpu": torch.cuda.get_device_name(dev)}
    print(json.dumps(res))
    if args.json:
        Path(args.json).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
