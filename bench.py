"""Benchmark: FFA fwd+bwd mask-aware TFLOPS on MAGI-1 block-causal masks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl magi|reference]

N=1 workload = BASELINE.json configs[1]: MAGI-1 4.5B attention layer
(24 query heads, 8 key/value heads, head_dim 128), bf16, 8 chunks of 4096
tokens block-causal (S = 32768). One step = FFA forward + backward
(preprocess, dK/dV pass, dQ pass) over that layer. FLOPs follow the
reference's mask-aware count (proj/src/sim.cpp:29-34): fwd = 4 * area_mult *
hq * d, bwd = fwd * 5 / 2.

N>1 runs the context-parallel path (cp.py): weak scaling, 131072 tokens per
rank, MAGI-1 24B shape, block 8192, one process per
GPU under torchrun; `value` is whole-job TFLOPS (total FLOPs / max-over-ranks
device time).

`--impl reference` times the CPU oracle port (oracle/ffa_oracle.c — the
reference has no attention arithmetic of its own) on a bounded
sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FFA fwd+bwd mask-aware TFLOPS (block-causal) and CP tokens/s at 1/2/4/8 B200"
UNIT = "TFLOPS"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"bf16": d.get("bf16_tflops", 1590.0), "bf16_sustained": d.get("bf16_tflops_sustained"),
                "source": "measured"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback"}


def block_causal(seqlen: int, block: int):
    qr = [[b, b + block] for b in range(0, seqlen, block)]
    kr = [[0, b + block] for b in range(0, seqlen, block)]
    return qr, kr, [0] * len(qr)


def block_causal_area(seqlen: int, block: int) -> int:
    n = seqlen // block
    return n * (n + 1) // 2 * block * block


def varlen_packed(seqlen: int, seed: int = 42, median: float = 2048.0, sigma: float = 1.0):
    """BASELINE configs[3] / SURVEY §8d config 4: sample lengths from the
    reference's deterministic log-normal generator (proj/src/pack.cpp:228-253,
    reimplemented bit-exactly in the planner), taken in order until they cover
    `seqlen`, the last one clipped; even samples FULL, odd samples CAUSAL."""
    from paper_2505_13211_b200.planner import lognormal_lengths

    lens, total, n = [], 0, 64
    while total < seqlen:
        lens = lognormal_lengths(n, median, sigma, seqlen, seed)
        total = sum(lens)
        n *= 2
    out, acc = [], 0
    for x in lens:
        x = min(x, seqlen - acc)
        out.append(x)
        acc += x
        if acc == seqlen:
            break
    qr, kr, ty, off = [], [], [], 0
    for i, n_ in enumerate(out):
        qr.append([off, off + n_])
        kr.append([off, off + n_])
        ty.append(0 if i % 2 == 0 else 1)
        off += n_
    return qr, kr, ty


WORKLOADS = {
    # BASELINE.json configs[1]
    "magi1_4.5b_layer_s32k_b4096": dict(seqlen=32768, hq=24, hk=8, d=128, block=4096),
    # BASELINE.json configs[2]
    "magi1_24b_layer_s32k_b4096": dict(seqlen=32768, hq=48, hk=8, d=128, block=4096),
    # BASELINE.json configs[3]: varlen packed FULL/CAUSAL clips
    "varlen_packed_s32k": dict(seqlen=32768, hq=48, hk=8, d=128, block=4096, varlen=True),
}
DEFAULT_WORKLOAD = "magi1_4.5b_layer_s32k_b4096"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


class EnergyMeter:
    """NVML's total-energy counter (mJ) read on both sides of the timed
    region: joules per step and mean board power under the power cap. None
    when NVML is unavailable; it never fails the bench."""

    def __init__(self, gpu: int):
        self.h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
        except Exception:  # noqa: BLE001
            self.h = None
        self.e0 = self.t0 = None

    def _read(self):
        if self.h is None:
            return None
        try:
            return float(self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h))
        except Exception:  # noqa: BLE001
            return None

    def start(self):
        self.e0, self.t0 = self._read(), time.perf_counter()

    def stop(self, steps: int) -> dict | None:
        e1, t1 = self._read(), time.perf_counter()
        if self.e0 is None or e1 is None or e1 <= self.e0 or steps <= 0:
            return None
        joules = (e1 - self.e0) * 1e-3
        return {"j_per_step": joules / steps, "avg_w": joules / (t1 - self.t0),
                "source": "NVML total energy counter around the timed region (host-clocked)"}


def cpu_baseline_sample(wl: dict, target_s: float = 12.0) -> dict:
    """Oracle port (oracle/ffa_oracle.c) fwd (f32 accumulate) + bwd on a bounded
    sample of the workload: the first `rows` query rows of chunk 0 against its
    whole key block, all heads. Timed on all host threads."""
    import numpy as np

    from oracle import oracle

    d, hq, hk, block = wl["d"], wl["hq"], wl["hk"], wl["block"]
    rng = np.random.default_rng(0)

    def run(rows: int) -> tuple[float, int]:
        q = rng.standard_normal((rows, hq, d), dtype=np.float32)
        k = rng.standard_normal((block, hk, d), dtype=np.float32)
        v = rng.standard_normal((block, hk, d), dtype=np.float32)
        do = rng.standard_normal((rows, hq, d), dtype=np.float32)
        qr, kr, ty = [[0, rows]], [[0, block]], [0]
        scale = 1.0 / math.sqrt(d)
        t0 = time.perf_counter()
        o, lse = oracle.ffa_fwd(q, k, v, qr, kr, ty, scale, acc_f32=True)
        oracle.ffa_bwd(q, k, v, o, lse, do, qr, kr, ty, scale)
        dt = time.perf_counter() - t0
        area = rows * block
        flops = 4 * area * hq * d
        return dt, flops + flops * 5 // 2

    rows = 16
    dt, fl = run(rows)
    rows = int(max(16, min(block, rows * target_s / max(dt, 1e-3))))
    dt, fl = run(rows)
    return {"value": fl / dt / 1e12, "unit": UNIT, "cores": oracle.num_threads(), "kind": "port",
            "sample": f"fwd(f32 acc)+bwd(f64) of {rows} query rows x {block} keys (full slice of "
                      f"chunk 0), {hq} q heads / {hk} kv heads, d={d}; {dt:.1f} s",
            "seconds": dt}


def host_info() -> dict:
    model = ""
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def planner_timing(reps: int = 3) -> dict:
    """The reference's own CPU path for CP planning (mask
    sweep, greedy dispatch, KV demands, transfer tables, stage solve), timed
    on this host through magiplan_scenario_parse + magiplan_scenario_plan:
    the reference compiled from its sources (oracle/_ref, test
    infrastructure) beside this library, plan JSON compared byte for byte.
    Single-threaded, as the reference is."""
    from tools import bench_planner as bp

    if not bp.REF.exists():
        return {"unavailable": "oracle/_ref/libmagiplan_ref.so not built"}
    ours, ref = bp._bind(bp.OURS), bp._bind(bp.REF)
    rows = []
    for name, spec in bp.scenarios():
        if "S=1048576 cp=8 block=8192" not in name and "S=524288" not in name and "S=131072" not in name:
            continue
        t_ours, ms_ours = bp._plan(ours, spec, reps)
        t_ref, ms_ref = bp._plan(ref, spec, reps)
        rows.append({"scenario": name, "reference_ms": round(statistics.median(ms_ref), 2),
                     "ours_ms": round(statistics.median(ms_ours), 2), "identical_plan_json": t_ours == t_ref})
    return {"what": "scenario_plan (shard + greedy + demands + tables + solve), 1 thread",
            "cores": 1, **host_info(), "runs": rows}


def single_config(workload: str) -> tuple[dict, tuple]:
    """The N=1 line's `config` (shared by both arms) and the slice list."""
    from paper_2505_13211_b200.planner import Mask

    wl = WORKLOADS[workload]
    S, hq, hk, d, block = wl["seqlen"], wl["hq"], wl["hk"], wl["d"], wl["block"]
    if wl.get("varlen"):
        qr, kr, ty = varlen_packed(S)
        mask_desc = f"varlen packed FULL/CAUSAL, {len(qr)} samples (lognormal median 2048, sigma 1, seed 42)"
    else:
        qr, kr, ty = block_causal(S, block)
        mask_desc = f"block_causal(block={block})"
    names = {0: "full", 1: "causal", 2: "inv_causal", 3: "bi_causal"}
    area = Mask({"seqlen_q": S, "seqlen_k": S, "slices": [{"q": a, "k": b, "type": names[t]}
                                                           for a, b, t in zip(qr, kr, ty)]}).area()
    fwd = 4 * area * hq * d
    cfg = {"workload": workload, "seqlen": S, "num_heads_q": hq, "num_heads_k": hk, "head_dim": d,
           "mask": mask_desc, "area_multiplicity": area, "flops_per_step": fwd + fwd * 5 // 2,
           "parallelism": "single GPU",
           "l2": f"inputs larger than L2 (q {S * hq * d * 2 / 1e6:.0f} MB, dO {S * hq * d * 2 / 1e6:.0f} MB "
                 f"> 126 MB); no flush"}
    return cfg, (qr, kr, ty)


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # all the host's threads for the CPU path: torchrun exports
    # OMP_NUM_THREADS=1 to every rank, and the oracle shares torch's OpenMP
    # runtime, so reset both before the first parallel region
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    wl = WORKLOADS[args.workload]
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    if world > 1:
        # the N>1 arm's workload: the CP config-5 shape (cp_bench), per-rank
        # tokens x N, block-causal 8192; the CPU sample is bounded either way
        from paper_2505_13211_b200 import cp_bench

        wl = dict(seqlen=cp_bench.PER_RANK * world, hq=cp_bench.HQ, hk=cp_bench.HK, d=cp_bench.D,
                  block=cp_bench.BLOCK)
        config = cp_bench.config(world, args.cp_mode)
    else:
        config, _ = single_config(args.workload)
    for _ in range(args.warmup):
        cpu_baseline_sample(wl, target_s=2.0)
    vals, samples = [], []
    for _ in range(args.steps):
        r = cpu_baseline_sample(wl, target_s=6.0)
        vals.append(r["value"])
        samples.append(r)
    value = statistics.median(vals)
    base = samples[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": base["cores"], "kind": "port",
                         "sample": base["sample"], **host_info(), "reference_planner": planner_timing()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_single(args) -> None:
    import torch

    from paper_2505_13211_b200 import _lib
    from paper_2505_13211_b200.ffa import FFAPlan

    wl = WORKLOADS[args.workload]
    S, hq, hk, d, block = wl["seqlen"], wl["hq"], wl["hk"], wl["d"], wl["block"]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    config, (qr, kr, ty) = single_config(args.workload)
    plan = FFAPlan(qr, kr, ty, S, S, d)
    plan.prepare()
    area = plan.area()
    assert area == config["area_multiplicity"]
    if not wl.get("varlen"):
        assert area == block_causal_area(S, block)
    fwd_flops = 4 * area * hq * d
    bwd_flops = fwd_flops * 5 // 2
    step_flops = fwd_flops + bwd_flops

    g = torch.Generator(device="cpu").manual_seed(0)
    q_h = torch.randn(S, hq, d, generator=g).to(torch.bfloat16).pin_memory()
    k_h = torch.randn(S, hk, d, generator=g).to(torch.bfloat16).pin_memory()
    v_h = torch.randn(S, hk, d, generator=g).to(torch.bfloat16).pin_memory()
    do_h = torch.randn(S, hq, d, generator=g).to(torch.bfloat16).pin_memory()
    q, k, v, do = (t.to(dev) for t in (q_h, k_h, v_h, do_h))
    out = torch.empty(S, hq, d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(hq, S, dtype=torch.float32, device=dev)
    delta = torch.empty(hq, S, dtype=torch.float32, device=dev)
    dq = torch.empty(S, hq, d, dtype=torch.bfloat16, device=dev)
    dk = torch.empty(S, hk, d, dtype=torch.bfloat16, device=dev)
    dv = torch.empty(S, hk, d, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    L = _lib.lib()
    scale = 1.0 / math.sqrt(d)
    BF = _lib.BF16

    def fwd():
        _lib.check(L.magiplan_ffa_fwd(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                      out.data_ptr(), lse.data_ptr(), hq, hk, scale, BF, 0, sp))

    def pre():
        _lib.check(L.magiplan_ffa_bwd_preprocess(out.data_ptr(), do.data_ptr(), delta.data_ptr(),
                                                 S, hq, d, BF, sp))

    def dkdv():
        _lib.check(L.magiplan_ffa_bwd_dkdv(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                           lse.data_ptr(), delta.data_ptr(), do.data_ptr(),
                                           dk.data_ptr(), dv.data_ptr(), hq, hk, scale, BF, 0, sp))

    def dqp():
        _lib.check(L.magiplan_ffa_bwd_dq(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                         lse.data_ptr(), delta.data_ptr(), do.data_ptr(),
                                         dq.data_ptr(), hq, hk, scale, BF, 0, sp))

    parts = [("ffa_fwd", fwd, fwd_flops), ("bwd_preprocess", pre, 0),
             ("ffa_bwd_dkdv", dkdv, 8 * area * hq * d), ("ffa_bwd_dq", dqp, 2 * area * hq * d)]
    launches_per_step = 4

    for _ in range(args.warmup):
        for _, fn, _ in parts:
            fn()
    torch.cuda.synchronize()

    clocks = ClockSampler(0)
    clocks.start()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(parts) + 1)]
          for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    energy = EnergyMeter(0)
    torch.cuda.synchronize()
    energy.start()
    start.record(stream)
    for s in range(args.steps):
        ev[s][0].record(stream)
        for i, (_, fn, _) in enumerate(parts):
            fn()
            ev[s][i + 1].record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    step_energy = energy.stop(args.steps)
    total_ms = start.elapsed_time(end)
    per_part = {name: statistics.mean(ev[s][i].elapsed_time(ev[s][i + 1]) for s in range(args.steps))
                for i, (name, _, _) in enumerate(parts)}

    # e2e through the public API with host buffers: H2D of the step's inputs,
    # forward + backward, D2H of the gradients.
    o_h = torch.empty_like(out, device="cpu").pin_memory()
    dq_h = torch.empty_like(dq, device="cpu").pin_memory()
    dk_h = torch.empty_like(dk, device="cpu").pin_memory()
    dv_h = torch.empty_like(dv, device="cpu").pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (q_h, k_h, v_h, do_h))
    d2h = sum(t.numel() * t.element_size() for t in (o_h, dq_h, dk_h, dv_h))

    # Two device buffer sets so step i+1's inputs travel (H2D stream) and step
    # i-1's outputs return (D2H stream) while step i computes. Every step
    # still copies its own inputs in and its O, dQ, dK, dV out through PCIe.
    sets = [dict(q=q, k=k, v=v, do=do, out=out, dq=dq, dk=dk, dv=dv)]
    sets.append({n: torch.empty_like(t) for n, t in sets[0].items()})
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def step_on(b, ev_do, ev_fwd_done, ev_kv_done):
        _lib.check(L.magiplan_ffa_fwd(plan.handle, b["q"].data_ptr(), b["k"].data_ptr(), b["v"].data_ptr(),
                                      b["out"].data_ptr(), lse.data_ptr(), hq, hk, scale, BF, 0, sp))
        ev_fwd_done.record(stream)  # O can travel back while the backward computes
        stream.wait_event(ev_do)  # dO is only needed from the backward on
        _lib.check(L.magiplan_ffa_bwd_preprocess(b["out"].data_ptr(), b["do"].data_ptr(), delta.data_ptr(),
                                                 S, hq, d, BF, sp))
        _lib.check(L.magiplan_ffa_bwd_dkdv(plan.handle, b["q"].data_ptr(), b["k"].data_ptr(),
                                           b["v"].data_ptr(), lse.data_ptr(), delta.data_ptr(),
                                           b["do"].data_ptr(), b["dk"].data_ptr(), b["dv"].data_ptr(),
                                           hq, hk, scale, BF, 0, sp))
        ev_kv_done.record(stream)  # dK / dV can travel back while dQ computes
        _lib.check(L.magiplan_ffa_bwd_dq(plan.handle, b["q"].data_ptr(), b["k"].data_ptr(), b["v"].data_ptr(),
                                         lse.data_ptr(), delta.data_ptr(), b["do"].data_ptr(),
                                         b["dq"].data_ptr(), hq, hk, scale, BF, 0, sp))

    def e2e_run(n, start=None):
        mk = lambda: [torch.cuda.Event() for _ in range(n)]  # noqa: E731
        ev_qkv, ev_do, ev_fwd, ev_kv, ev_done, ev_out = mk(), mk(), mk(), mk(), mk(), mk()

        def h2d(i):
            b = sets[i % 2]
            with torch.cuda.stream(h2d_s):
                if i == 0 and start is not None:
                    h2d_s.wait_event(start)  # copies belong to the timed region
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
            stream.wait_event(ev_qkv[i])
            if i >= 2:
                stream.wait_event(ev_out[i - 2])  # gradients of this set already returned
            step_on(sets[i % 2], ev_do[i], ev_fwd[i], ev_kv[i])
            ev_done[i].record(stream)
            with torch.cuda.stream(d2h_s):
                b = sets[i % 2]
                d2h_s.wait_event(ev_fwd[i])
                o_h.copy_(b["out"], non_blocking=True)
                d2h_s.wait_event(ev_kv[i])
                dk_h.copy_(b["dk"], non_blocking=True)
                dv_h.copy_(b["dv"], non_blocking=True)
                d2h_s.wait_event(ev_done[i])
                dq_h.copy_(b["dq"], non_blocking=True)
                ev_out[i].record(d2h_s)
        stream.wait_event(ev_out[n - 1])

    e2e_run(2)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_run(args.steps, start=e0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()

    ms = total_ms / args.steps
    value = step_flops / (ms * 1e-3) / 1e12
    peaks = _peaks()
    kernels = {}
    for name, _, fl in parts:
        t = per_part[name]
        kernels[name] = {"ms": t, "share": t / sum(per_part.values()),
                         "tflops": (fl / (t * 1e-3) / 1e12) if fl else None}
    dom = max((n for n, _, fl in parts if fl), key=lambda n: per_part[n])
    dom_fl = dict((n, fl) for n, _, fl in parts)[dom]
    achieved = dom_fl / (per_part[dom] * 1e-3) / 1e12
    traffic, traffic_tag = None, None
    summ = ROOT / "profiles" / "ncu_summary.json"
    if summ.exists():
        try:
            js = json.loads(summ.read_text())
            traffic, traffic_tag = js.get("dram_bytes_per_launch", {}).get(dom), js.get("tag")
        except Exception:  # noqa: BLE001
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": config,
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peaks["bf16"],
                     "unit": "TFLOP/s", "frac": achieved / peaks["bf16"], "traffic": traffic,
                     "traffic_source": f"ncu --set full, profiles/ncu_{traffic_tag}.md" if traffic_tag else None,
                     "peak_source": peaks["source"], "peak_sustained": peaks["bf16_sustained"],
                     "step_frac": value / peaks["bf16"]},
        "kernels": kernels,
        "e2e": {"value": step_flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "copies": "H2D q, k, v, dO; D2H O, dQ, dK, dV (bf16), every step"},
        "clocks": clk,
        "energy": step_energy,
        "gpu_launches": launches_per_step * args.steps,
    }
    del sets, q, k, v, do, out, dq, dk, dv
    torch.cuda.empty_cache()
    if not args.no_weak_anchor:
        from paper_2505_13211_b200 import cp_bench

        line["weak_anchor"] = cp_bench.anchor(steps=2, warmup=1)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(wl)
        line["cpu_baseline"].pop("seconds", None)
        line["cpu_baseline"].update(host_info())
        line["cpu_baseline"]["reference_planner"] = planner_timing()
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="magi", choices=["magi", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-weak-anchor", action="store_true",
                    help="N=1: skip the cp=1 run of the CP weak-scaling workload")
    ap.add_argument("--cp-mode", default="magi", choices=["magi", "p2p", "capi", "capi_p2p", "ring", "ulysses"],
                    help="N>1 only: MagiAttention GroupCast CP (default; 'p2p' = the forward GroupCast "
                         "over NVLink peer memory instead of NCCL; 'capi' = the same schedule through the "
                         "C-ABI executor; 'capi_p2p' = that executor over NVLink peer memory), or the "
                         "ring-attention / Ulysses baselines")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1:
        from paper_2505_13211_b200 import cp_bench

        cp_bench.run(args)
        return
    run_single(args)


if __name__ == "__main__":
    main()
