"""C ABI boundary (CPU): exports, status mapping, error text, ownership.

Mirrors the reference's C ABI suite (proj/tests/test_capi.cpp:52-228):
status codes 2/3/4, thread-local last_error, byte-identical reruns across
jobs=1/2, and plan/simulate agreement."""
import ctypes as C
import json
import re
import threading
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> list[str]:
    text = (ROOT / "include" / "magiplan.h").read_text()
    return re.findall(r"MAGIPLAN_API\s+[\w\s\*]+?\b(magiplan_\w+)\s*\(", text)


def test_every_declared_symbol_is_exported(built_lib):
    from paper_2505_13211_b200 import _lib

    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(built_lib, n)]
    assert not missing, missing
    # the 14 reference entry points (magiplan.h:61-121) are all present
    ref14 = ["magiplan_version", "magiplan_last_error", "magiplan_string_free", "magiplan_mask_parse",
             "magiplan_mask_free", "magiplan_mask_area", "magiplan_mask_is_allowed",
             "magiplan_mask_render", "magiplan_mask_describe", "magiplan_scenario_parse",
             "magiplan_scenario_free", "magiplan_scenario_set_seed", "magiplan_scenario_plan",
             "magiplan_scenario_simulate", "magiplan_pack_run"]
    assert set(ref14) <= set(names)
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_version_and_status_mapping(built_lib):
    from paper_2505_13211_b200 import _lib

    L = built_lib
    assert L.magiplan_version() == b"0.1.0"
    h = C.c_void_p()
    assert L.magiplan_mask_parse(None, C.byref(h)) == _lib.ERR_USAGE
    assert L.magiplan_last_error() == b"null argument"
    assert L.magiplan_mask_parse(b"{not json", C.byref(h)) == _lib.ERR_USAGE
    assert b"mask spec" in L.magiplan_last_error()
    assert h.value is None  # outputs untouched on failure
    st = L.magiplan_mask_parse(b'{"seqlen": 10, "pattern": "block_causal", "params": {"block_size": 3}}',
                               C.byref(h))
    assert st == _lib.ERR_CONSTRAINT and b"does not divide" in L.magiplan_last_error()
    assert L.magiplan_mask_parse(b'{"seqlen": 8, "pattern": "causal"}', C.byref(h)) == _lib.OK
    assert L.magiplan_last_error() == b""  # success clears the error
    area = C.c_int64()
    assert L.magiplan_mask_area(h, _lib.COUNT_UNION, C.byref(area)) == _lib.OK and area.value == 36
    ok = C.c_int()
    assert L.magiplan_mask_is_allowed(h, 8, 0, C.byref(ok)) == _lib.ERR_USAGE
    L.magiplan_mask_free(h)


def test_last_error_is_thread_local(built_lib):
    from paper_2505_13211_b200 import _lib

    L = built_lib
    h = C.c_void_p()
    assert L.magiplan_mask_parse(b"[]", C.byref(h)) == _lib.ERR_USAGE
    seen = {}

    def other():
        seen["err"] = L.magiplan_last_error()

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen["err"] == b""
    assert L.magiplan_last_error() != b""


def test_scenario_reruns_identical_and_jobs_invariant(built_lib):
    from paper_2505_13211_b200.planner import Scenario

    spec = {"workload": {"mask": {"seqlen": 8192, "pattern": "full"}, "num_heads_q": 8},
            "sweep": {"cp_sizes": [1, 2, 4, 8], "per_rank_seqlen": 4096},
            "cost_model": {"ffa_fwd": {"latency": 1, "per_unit": 1e-4},
                           "cast": {"latency": 5, "per_unit": 0.01},
                           "reduce": {"latency": 5, "per_unit": 0.01},
                           "ffa_bwd": {"latency": 1, "per_unit": 2.5e-4}}}
    sc = Scenario(spec)
    a, b = sc.simulate_text(1), sc.simulate_text(2)
    assert a == b and len(a.strip().splitlines()) == 8
    sc.set_seed(9)
    assert all(json.loads(l)["seed"] == 9 for l in sc.simulate_text(1).splitlines())


def test_plan_and_simulate_agree(built_lib):
    """estimate == simulated makespan (reference test_sim.cpp:140-181)."""
    from paper_2505_13211_b200.planner import Scenario

    spec = {"workload": {"mask": {"seqlen": 16384, "pattern": "block_causal",
                                  "params": {"block_size": 2048}}},
            "cp_size": 4,
            "cost_model": {"ffa_fwd": {"latency": 30, "per_unit": 8.19e-05},
                           "ffa_bwd": {"latency": 30, "per_unit": 2.05e-04},
                           "cast": {"latency": 100, "per_unit": 0.082},
                           "reduce": {"latency": 100, "per_unit": 0.082}}}
    sc = Scenario(spec)
    plan = sc.plan()
    fwd, bwd = (json.loads(l) for l in sc.simulate_text().splitlines())
    est_f = max(r["est_cost_fwd"] for r in plan["overlap"]["ranks"])
    est_b = max(r["est_cost_bwd"] for r in plan["overlap"]["ranks"])
    assert fwd["makespan"] == est_f and bwd["makespan"] == est_b


def test_every_schedule_simulates(built_lib):
    """All five schedules of the reference simulator (sim.cpp:174-537) run
    through magiplan_scenario_simulate; magi/ring give fwd+bwd records,
    Ulysses/cso a forward record with its step log; errors map like the
    reference's (cso chunk count: USAGE, indivisible seqlen: CONSTRAINT)."""
    from paper_2505_13211_b200 import _lib
    from paper_2505_13211_b200.planner import Scenario

    def sim(schedule, seqlen=4096, cp=4, **extra):
        aff = lambda lat, pu: {"latency": lat, "per_unit": pu}  # noqa: E731
        cost = {"ffa_fwd": aff(30, 8.19e-05), "ffa_bwd": aff(30, 2.05e-04), "cast": aff(100, 0.082),
                "reduce": aff(100, 0.082), "q_proj": aff(10, 0.5), "k_proj": aff(10, 0.1),
                "v_proj": aff(10, 0.1), "kv_cache_update": aff(5, 0.05), "cross_attn": aff(10, 0.3)}
        spec = {"workload": {"mask": {"seqlen": seqlen, "pattern": "causal"}}, "cp_size": cp,
                "schedule": schedule, "cost_model": cost, **extra}
        return [json.loads(l) for l in Scenario(spec).simulate_text().splitlines()]

    for sched, passes in (("magi", ["fwd", "bwd"]), ("ring", ["fwd", "bwd"]),
                          ("ring_serial", ["fwd", "bwd"]), ("ulysses", ["fwd"]), ("cso", ["fwd"])):
        recs = sim(sched)
        assert [r["pass"] for r in recs] == passes and all(r["schedule"] == sched for r in recs)
        assert all(r["makespan"] > 0 and len(r["per_rank_makespan"]) == 4 for r in recs)
    # overlapping the ring hops never loses to the serial ring
    assert sim("ring")[0]["makespan"] <= sim("ring_serial")[0]["makespan"]
    assert len(sim("cso", cso_num_chunks=3)[0]["event_log"]) == 3 + 3
    with pytest.raises(_lib.UsageError):
        sim("cso", cso_num_chunks=1)
    with pytest.raises(_lib.ConstraintError):
        sim("ulysses", seqlen=4098)


def test_ffa_plan_validation_on_cpu(built_lib):
    """Plan construction is host-only until upload; bad slices are USAGE errors."""
    from paper_2505_13211_b200 import _lib

    L = built_lib
    qr = (C.c_int64 * 2)(0, 300)
    kr = (C.c_int64 * 2)(0, 100)
    ty = (C.c_int32 * 1)(0)
    h = C.c_void_p()
    st = L.magiplan_ffa_plan_create(qr, kr, ty, 1, 200, 200, 128, C.byref(h))
    assert st == _lib.ERR_USAGE and b"exceeds mask bounds" in L.magiplan_last_error()
    st = L.magiplan_ffa_plan_create(qr, kr, ty, 1, 300, 300, 96, C.byref(h))
    assert st == _lib.ERR_USAGE and b"head_dim" in L.magiplan_last_error()


def test_cp_create_argument_validation_on_cpu(built_lib):
    """The CP executor rejects a bad transport / head layout before touching
    CUDA or NCCL (USAGE error, handle untouched)."""
    from paper_2505_13211_b200 import _lib
    from paper_2505_13211_b200.planner import Scenario

    L = built_lib
    sc = Scenario({"workload": {"mask": {"seqlen": 4096, "pattern": "causal"}, "num_heads_q": 4,
                                "num_heads_k": 2, "head_dim": 128}, "cp_size": 2})
    uid = C.create_string_buffer(128)
    h = C.c_void_p()
    st = L.magiplan_cp_create_ex(sc._h, 0, uid, 4, 2, 128, 0.088, 7, C.byref(h))
    assert st == _lib.ERR_USAGE and b"transport" in L.magiplan_last_error() and h.value is None
    st = L.magiplan_cp_create_ex(sc._h, 0, uid, 4, 3, 128, 0.088, 1, C.byref(h))
    assert st == _lib.ERR_USAGE and b"multiple of num_heads_k" in L.magiplan_last_error()
    st = L.magiplan_cp_create_ex(sc._h, 0, uid, 4, 2, 96, 0.088, 0, C.byref(h))
    assert st == _lib.ERR_USAGE and b"head_dim" in L.magiplan_last_error()


# ---------------------------------------------------------------- a plain C consumer
def _build_c_consumer() -> Path:
    """gcc-compile tests/c_consumer/ffa_consumer.c against include/ and the
    in-tree libmagiplan.so (+ the CUDA runtime for its device buffers): the
    link a C client of the reference planner does after the switch."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    cuda = Path("/usr/local/cuda")
    out = ROOT / "build" / "c_consumer" / "ffa_consumer"
    out.parent.mkdir(parents=True, exist_ok=True)
    pkg = ROOT / "paper_2505_13211_b200"
    cmd = ["gcc", "-O2", "-std=c11", str(ROOT / "tests" / "c_consumer" / "ffa_consumer.c"),
           f"-I{ROOT / 'include'}", f"-I{cuda / 'include'}", f"-L{pkg}", "-lmagiplan",
           f"-L{cuda / 'lib64'}", "-lcudart", "-lm", f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{cuda / 'lib64'}",
           "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return out


def test_c_consumer_planner(built_lib):
    """The reference's own entry points called from C (no Python in the
    process): the mask area and the scenario plan match the ctypes path."""
    import subprocess

    from paper_2505_13211_b200 import _lib
    from paper_2505_13211_b200.planner import Mask, Scenario

    exe = _build_c_consumer()
    res = subprocess.run([str(exe), "plan"], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    area, nbytes = (int(x) for x in res.stdout.split()[1::2])
    assert area == Mask({"seqlen": 32768, "pattern": "block_causal", "params": {"block_size": 4096}}).area()
    scen = {"workload": {"mask": {"seqlen": 131072, "pattern": "block_causal", "params": {"block_size": 8192}},
                         "num_heads_q": 48, "num_heads_k": 8, "num_heads_v": 8, "head_dim": 128},
            "cp_size": 4}
    assert nbytes == len(Scenario(scen).plan_text().encode())
    assert _lib is not None


def _xorshift_bf16(n: int, state: list[int]):
    """The consumer's input stream (xorshift32 -> uniform [-1, 1) -> bf16,
    round to nearest even), regenerated bit for bit."""
    import numpy as np

    out = np.empty(n, np.float32)
    s = state[0]
    for i in range(n):
        s ^= (s << 13) & 0xFFFFFFFF
        s ^= s >> 17
        s ^= (s << 5) & 0xFFFFFFFF
        out[i] = np.float32((s >> 8) / 16777216.0 * 2.0 - 1.0)
    state[0] = s
    u = out.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.gpu
def test_c_consumer_ffa_matches_oracle(built_lib, cuda, tmp_path):
    """FFA forward + backward driven from C through the ABI (cudaMalloc'd
    buffers, a cudaStream_t, no torch in the process), checked against the
    CPU oracle on the same inputs: 640 tokens, block-causal 128 plus an
    overlapping causal slice, 4 q / 2 kv heads, d = 128, f32 outputs."""
    import math
    import subprocess

    import numpy as np
    from oracle import oracle

    exe = _build_c_consumer()
    path = tmp_path / "ffa.bin"
    res = subprocess.run([str(exe), "ffa", str(path)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    S, HQ, HK, D = 640, 4, 2, 128
    qr = [[0, 128], [128, 256], [256, 384], [384, 512], [512, 640], [0, 200]]
    kr = [[0, 128], [0, 256], [0, 384], [0, 512], [0, 640], [0, 200]]
    ty = [0, 0, 0, 0, 0, 1]
    st = [12345]
    q = _xorshift_bf16(S * HQ * D, st).reshape(S, HQ, D)
    k = _xorshift_bf16(S * HK * D, st).reshape(S, HK, D)
    v = _xorshift_bf16(S * HK * D, st).reshape(S, HK, D)
    do = _xorshift_bf16(S * HQ * D, st).reshape(S, HQ, D)
    raw = np.fromfile(path, np.float32)
    sizes = [S * HQ * D, HQ * S, S * HQ * D, S * HK * D, S * HK * D]
    parts, off = [], 0
    for n in sizes:
        parts.append(raw[off:off + n])
        off += n
    o, lse, dq, dk, dv = parts
    scale = 1.0 / math.sqrt(D)
    ro, rl = oracle.ffa_fwd(q, k, v, qr, kr, ty, scale)
    rdq, rdk, rdv = oracle.ffa_bwd(q, k, v, ro, rl, do, qr, kr, ty, scale)

    def rel(a, b):
        return float(np.abs(a - b).max() / np.abs(b).max())

    assert rel(o.reshape(ro.shape), ro) < 5e-3
    assert float(np.abs(lse.reshape(rl.shape) - rl).max()) < 2e-4
    for got, ref in ((dq, rdq), (dk, rdk), (dv, rdv)):
        assert rel(got.reshape(ref.shape), ref) < 1e-2
