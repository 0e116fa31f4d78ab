"""bench.py's host-side contract pieces, on CPU: the shared `config` of both
arms at every N, the workloads' FLOP accounting against the planner, and the
guarded measurement helpers (they never fail the bench)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def test_energy_meter_is_guarded():
    import bench

    m = bench.EnergyMeter(0)
    m.start()
    e = m.stop(3)
    # null without NVML / a GPU; otherwise joules per step and mean power
    assert e is None or (e["j_per_step"] > 0 and e["avg_w"] > 0)
    assert bench.EnergyMeter(0).stop(0) is None


@pytest.mark.parametrize("workload", ["magi1_4.5b_layer_s32k_b4096", "magi1_24b_layer_s32k_b4096",
                                      "varlen_packed_s32k"])
def test_single_config_area_and_flops_closed_form(built_lib, workload):
    import bench

    cfg, (qr, kr, ty) = bench.single_config(workload)
    wl = bench.WORKLOADS[workload]
    S = wl["seqlen"]
    if wl.get("varlen"):
        # documents back to back: FULL n^2 pairs, CAUSAL n(n+1)/2
        lens = [b - a for a, b in qr]
        assert sum(lens) == S and [list(x) for x in qr] == [list(x) for x in kr]
        area = sum(n * n if t == 0 else n * (n + 1) // 2 for n, t in zip(lens, ty))
    else:
        area = bench.block_causal_area(S, wl["block"])
    assert area == cfg["area_multiplicity"]
    fwd = 4 * cfg["area_multiplicity"] * wl["hq"] * wl["d"]
    assert cfg["flops_per_step"] == fwd + fwd * 5 // 2  # reference sim.cpp:29-34
    assert cfg["workload"] == workload


@pytest.mark.parametrize("world", [2, 4, 8])
def test_cp_config_same_keys_every_mode(built_lib, world):
    from paper_2505_13211_b200 import cp_bench

    cfgs = {m: cp_bench.config(world, m) for m in ("magi", "p2p", "capi", "capi_p2p", "ring", "ulysses")}
    keys = {tuple(sorted(c)) for c in cfgs.values()}
    assert len(keys) == 1
    # the work is the same whatever the transport or CP mode
    assert len({c["flops_per_step"] for c in cfgs.values()}) == 1
    assert cfgs["magi"]["parallelism"] == f"cp{world}"


def test_cli_lists_every_cp_mode():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120, check=True).stdout
    for mode in ("magi", "p2p", "capi", "capi_p2p", "ring", "ulysses"):
        assert mode in out
