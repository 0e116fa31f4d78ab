"""Planner timing, this library vs the reference.

Both libraries are driven through the identical C ABI
(magiplan_scenario_parse + magiplan_scenario_plan: mask sweep, dispatch,
KV demands, transfer tables, overlap-stage solve, plan JSON) on the same
scenarios; the reference is the planner compiled from its own sources by
oracle/Makefile (oracle/_ref/libmagiplan_ref.so, test infrastructure). The
plan JSON must be byte-identical; the wall time per plan is reported.

    python tools/bench_planner.py            # prints one JSON line per scenario
"""
from __future__ import annotations

import ctypes as C
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OURS = ROOT / "paper_2505_13211_b200" / "libmagiplan.so"
REF = ROOT / "oracle" / "_ref" / "libmagiplan_ref.so"

COST = {"ffa_fwd": {"latency": 30, "per_unit": 8.19e-05}, "ffa_bwd": {"latency": 30, "per_unit": 2.05e-04},
        "cast": {"latency": 100, "per_unit": 0.082}, "reduce": {"latency": 100, "per_unit": 0.082}}


def scenarios():
    for S, cp, block in ((131072, 2, 8192), (524288, 4, 8192), (1048576, 8, 8192), (1048576, 8, 32768)):
        yield f"block_causal S={S} cp={cp} block={block}", {
            "workload": {"mask": {"seqlen": S, "pattern": "block_causal", "params": {"block_size": block}},
                         "batch_size": 1, "num_heads_q": 48, "num_heads_k": 8, "num_heads_v": 8,
                         "head_dim": 128, "dtype_bytes": 2},
            "schedule": "magi", "cp_size": cp, "dispatch": "greedy", "dispatch_chunk_size": S // cp // 8,
            "cost_model": COST, "overlap": {"min_chunk_size": 512, "max_num_chunks": 8}, "seed": 0}
    yield "causal S=1048576 cp=8", {
        "workload": {"mask": {"seqlen": 1048576, "pattern": "causal"}, "batch_size": 1, "num_heads_q": 48,
                     "num_heads_k": 8, "num_heads_v": 8, "head_dim": 128, "dtype_bytes": 2},
        "schedule": "magi", "cp_size": 8, "dispatch": "greedy", "dispatch_chunk_size": 16384,
        "cost_model": COST, "overlap": {"min_chunk_size": 512, "max_num_chunks": 8}, "seed": 0}


def _bind(path: Path):
    lib = C.CDLL(str(path))
    lib.magiplan_scenario_parse.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
    lib.magiplan_scenario_parse.restype = C.c_int
    lib.magiplan_scenario_plan.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.magiplan_scenario_plan.restype = C.c_int
    lib.magiplan_scenario_free.argtypes = [C.c_void_p]
    lib.magiplan_string_free.argtypes = [C.c_void_p]
    lib.magiplan_last_error.restype = C.c_char_p
    return lib


def _plan(lib, spec: dict, reps: int) -> tuple[str, list[float]]:
    sc = C.c_void_p()
    if lib.magiplan_scenario_parse(json.dumps(spec).encode(), b".", C.byref(sc)) != 0:
        raise RuntimeError(lib.magiplan_last_error().decode())
    times, text = [], ""
    try:
        for _ in range(reps):
            out = C.c_void_p()
            t0 = time.perf_counter()
            st = lib.magiplan_scenario_plan(sc, C.byref(out))
            times.append((time.perf_counter() - t0) * 1e3)
            if st != 0:
                raise RuntimeError(lib.magiplan_last_error().decode())
            text = C.string_at(out.value).decode()
            lib.magiplan_string_free(out)
    finally:
        lib.magiplan_scenario_free(sc)
    return text, times


def main(reps: int = 3) -> None:
    if not REF.exists():
        print(json.dumps({"unavailable": f"{REF} missing (build with make -C oracle ref)"}))
        return
    ours, ref = _bind(OURS), _bind(REF)
    for name, spec in scenarios():
        t_ours, ms_ours = _plan(ours, spec, reps)
        t_ref, ms_ref = _plan(ref, spec, reps)
        print(json.dumps({"scenario": name, "identical_plan_json": t_ours == t_ref,
                          "ours_ms": round(statistics.median(ms_ours), 2),
                          "reference_ms": round(statistics.median(ms_ref), 2),
                          "speedup": round(statistics.median(ms_ref) / statistics.median(ms_ours), 2)}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
