"""Planner parity (CPU): every golden record produced by the compiled
reference planner (oracle/ref_golden.cpp -> tests/golden/ref_planner.json)
is replayed through libmagiplan.so and must agree exactly: integer areas,
slice lists, dispatch assignments, demand sets, transfer tables, package /
stage plans, and byte-identical plan / simulate JSON."""
import json
from pathlib import Path

import pytest

GOLD = json.loads((Path(__file__).parent / "golden" / "ref_planner.json").read_text())


@pytest.fixture(scope="module")
def P(built_lib):
    from paper_2505_13211_b200 import planner

    return planner


def test_slice_area(P):
    for s, area in GOLD["slice_area"]:
        assert P.debug_eval("slice_area", slice=s) == area, s


def test_slice_area_in_cols(P):
    for s, cols, area in GOLD["slice_area_in_cols"]:
        assert P.debug_eval("slice_area_in_cols", slice=s, cols=cols) == area, (s, cols)


def test_named_masks(P):
    for e in GOLD["named_masks"]:
        got = P.debug_eval("mask", mask=e["spec"], rows="row_counts" in e)
        assert got["json"] == e["json"]
        assert got["area_union"] == e["area_union"]
        assert got["area_multiplicity"] == e["area_multiplicity"]
        if "row_counts" in e:
            assert got["row_counts"] == e["row_counts"]
        if "ascii" in e:
            assert P.Mask(e["spec"]).render() == e["ascii"]


def test_random_masks_union_and_restrict(P):
    for e in GOLD["random_masks"]:
        got = P.debug_eval("mask", mask=e["mask"], rows=True)
        assert got["area_union"] == e["area_union"]
        assert got["area_multiplicity"] == e["area_multiplicity"]
        assert got["row_counts"] == e["row_counts"]
        assert P.debug_eval("restrict_rows", mask=e["mask"], rows=e["rows"]) == e["restricted"]


def test_dispatch_bit_exact(P):
    for e in GOLD["dispatch"]:
        for op in ("greedy", "zigzag", "brute_force"):
            if op in e:
                assert P.debug_eval(op, areas=e["areas"], cp=e["cp"]) == e[op], (op, e["areas"], e["cp"])


def test_demands_and_tables(P):
    for e in GOLD["demands"]:
        assert P.debug_eval("shard", mask=e["mask"], chunk=e["chunk"]) == e["chunk_areas"]
        got = P.debug_eval("demands", mask=e["mask"], chunk=e["chunk"], cp=e["cp"],
                           assignment=e["assignment"])
        assert got["demands"] == e["demands"]
        assert got["cast"] == e["cast"]
        assert got["reduce"] == e["reduce"]
        assert got["redundancy"] == e["redundancy"]


def test_overlap_pieces(P):
    for tr, mn, mx, want in GOLD["partition_packages"]:
        assert P.debug_eval("partition_packages", traffic=tr, min=mn, max=mx) == want
    for e in GOLD["assign_packages"]:
        assert P.debug_eval("assign_packages", sizes=e["sizes"], stages=e["stages"]) == e["lpt"]
        if "seed" in e:
            got = P.debug_eval("assign_packages", sizes=e["sizes"], stages=e["stages"], seed=e["seed"])
            assert got == e["shuffled"]
    for e in GOLD["estimates"]:
        assert P.debug_eval("estimate", host=e["host"], compute=e["compute"], cast=e["cast"],
                            reduce=e["reduce"]) == [e["fwd"], e["bwd"]]
    for e in GOLD["fit_affine"]:
        assert P.debug_eval("fit_affine", samples=e["samples"]) == pytest.approx(e["fit"], rel=0, abs=0)


def test_lognormal_lengths(P):
    assert P.lognormal_lengths(200, 2048.0, 1.0, 65536, 42) == GOLD["lognormal_2048_1.0_65536_seed42"]


def test_flops(P):
    got = P.debug_eval("flops", mask={"seqlen": 4096, "pattern": "full"}, num_heads_q=64, head_dim=128)
    assert got == GOLD["flops_full4096_h64_d128"] == [549755813888, 1374389534720]


@pytest.mark.parametrize("idx", range(len(GOLD["scenarios"])))
def test_scenarios_byte_identical(P, idx):
    from paper_2505_13211_b200 import _lib

    e = GOLD["scenarios"][idx]
    text = e["scenario"]
    try:
        sc = P.Scenario(text)
    except _lib.MagiplanError as err:
        assert e.get("plan", "").startswith("ERROR") or e.get("simulate", "").startswith("ERROR")
        want = (e.get("plan") or e["simulate"])[len("ERROR "):]
        assert err.message == want
        return
    if "plan" in e:
        if e["plan"].startswith("ERROR"):
            with pytest.raises(_lib.MagiplanError) as ei:
                sc.plan_text()
            assert ei.value.message == e["plan"][len("ERROR "):]
        else:
            assert sc.plan_text() == e["plan"]
    if "simulate" in e:
        if e["simulate"].startswith("ERROR"):
            with pytest.raises(_lib.MagiplanError) as ei:
                sc.simulate_text(2)
            assert ei.value.message == e["simulate"][len("ERROR "):]
        else:
            assert sc.simulate_text(2) == e["simulate"]


@pytest.mark.parametrize("idx", range(len(GOLD["pack_runs"])))
def test_pack_run_byte_identical(P, idx):
    """magiplan_pack_run against the reference library's report, byte for
    byte; errors by class and message (reference capi.cpp:188-198,
    scenario.cpp:428-554, pack.cpp:30-226)."""
    from paper_2505_13211_b200 import _lib

    e = GOLD["pack_runs"][idx]
    if e["out"].startswith("ERROR "):
        with pytest.raises(_lib.MagiplanError) as ei:
            P.pack_run_text(e["config"], e.get("stream"))
        assert ei.value.message == e["out"][len("ERROR "):]
        kind = _lib.ConstraintError if "constraint violated" in e["out"] else _lib.UsageError
        assert isinstance(ei.value, kind)
    else:
        assert P.pack_run_text(e["config"], e.get("stream")) == e["out"]


def test_pack_invariants(P):
    """Every emitted bin fits max_length and is non-empty, each sample is
    packed at most once, and the counts balance (reference pack.cpp:135-196)."""
    lengths = P.lognormal_lengths(3000, 2048.0, 1.0, 32768, 42)
    cfg = {"packing": {"max_length": 32768, "bins_per_iteration": 8, "pool_capacity": 64, "dp_size": 4},
           "emit_bins": True}
    stream = "".join(f"{i} {n}\n" for i, n in enumerate(lengths))
    rep = P.pack_run(cfg, stream)
    seen = set()
    for batch in rep["batches"]:
        assert len(batch["bins"]) == 8
        for b in batch["bins"]:
            assert b["samples"] and b["fill"] == sum(s["length"] for s in b["samples"]) <= 32768
            for s in b["samples"]:
                assert s["id"] not in seen and lengths[s["id"]] == s["length"]
                seen.add(s["id"])
    assert rep["samples_packed"] == len(seen)
    assert rep["samples_packed"] + rep["samples_left"] + rep["skipped_oversized"] == rep["samples_in"]
    assert rep["stats"]["min_utilization"] >= 0.5  # the default defer_threshold
    docs = P.pack_samples(lengths[:200], 32768, 2)
    assert all(sum(d) <= 32768 for d in docs)


def test_packed_bin_masks(P):
    """Packer output as FFA masks: documents back to back, padding tail
    without slices, MULTIPLICITY area = sum of per-document areas."""
    lengths = P.lognormal_lengths(400, 2048.0, 1.0, 16384, 7)
    masks = P.packed_bin_masks(lengths, 16384, 4)
    assert masks
    for spec in masks:
        m = P.Mask(spec)
        want, end = 0, 0
        for i, (q, k, ty) in enumerate(m.slices):
            n = q[1] - q[0]
            assert q == k and q[0] == end and ty == (1 if i % 2 else 0)
            want += n * n if ty == 0 else n * (n + 1) // 2
            end = q[1]
        assert end <= 16384 and m.area() == want == m.area(union=True)
