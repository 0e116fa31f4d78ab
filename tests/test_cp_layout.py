"""Context-parallel host logic on CPU.

1. The executor plan (magiplan_scenario_exec_plan) re-expresses each rank's
   local mask exactly: host slices over local KV plus every stage's slices
   over its receive buffer, mapped back to global coordinates, equal the
   rank's rows of the global mask pair-for-pair with multiplicity.
2. The GroupCast / GroupReduce exchange pattern built from it moves exactly
   the right tokens, run with the gloo backend at world size 2, 4 and 8 (the
   NCCL path on GPUs uses the same layouts).
"""
import json
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

COST = {"ffa_fwd": {"latency": 30, "per_unit": 8.19e-05}, "ffa_bwd": {"latency": 30, "per_unit": 2.05e-04},
        "cast": {"latency": 100, "per_unit": 0.082}, "reduce": {"latency": 100, "per_unit": 0.082}}

MASKS = [
    ({"seqlen": 256, "pattern": "block_causal", "params": {"block_size": 32}}, 4, 8),
    ({"seqlen": 240, "pattern": "causal"}, 3, 10),
    ({"seqlen": 192, "pattern": "sliding_window_causal", "params": {"window": 20}}, 4, 6),
    ({"seqlen": 256, "pattern": "varlen_block_causal_last_global",
      "params": {"sample_lengths": [128, 64, 64], "block_size": 16}}, 2, 16),
    ({"seqlen_q": 160, "seqlen_k": 160, "slices": [
        {"q": [0, 100], "k": [0, 160], "type": "inv_causal"},
        {"q": [40, 160], "k": [10, 150], "type": "bi_causal"},
        {"q": [0, 160], "k": [30, 90], "type": "causal"}]}, 4, 5),
    # cp 8 (the 1M-token bench shape, scaled down): 64 chunks, 8 per rank
    ({"seqlen": 512, "pattern": "block_causal", "params": {"block_size": 64}}, 8, 8),
]


# A cost model under which splitting is free and the cast is expensive: the
# overlap solver then takes as many stages as there are packages, so
# `max_num_chunks` forces the stage count (Alg. 2, overlap.cpp:343-399).
COST_STAGED = {"ffa_fwd": {"latency": 0, "per_unit": 8.19e-05}, "ffa_bwd": {"latency": 0, "per_unit": 2.05e-04},
               "cast": {"latency": 0, "per_unit": 0.082}, "reduce": {"latency": 0, "per_unit": 0.082}}


def scenario(mask, cp, chunk, min_chunk=16, max_chunks=5, stages=None):
    """stages=None: the default cost model (one stage on these sizes);
    stages=s: COST_STAGED with s packages, i.e. up to s fwd / bwd stages."""
    if stages is not None:
        return {"workload": {"mask": mask, "num_heads_q": 4, "num_heads_k": 2}, "cp_size": cp,
                "dispatch_chunk_size": chunk, "cost_model": COST_STAGED,
                "overlap": {"min_chunk_size": 4, "max_num_chunks": stages}}
    return {"workload": {"mask": mask, "num_heads_q": 4, "num_heads_k": 2}, "cp_size": cp,
            "dispatch_chunk_size": chunk, "cost_model": COST,
            "overlap": {"min_chunk_size": min_chunk, "max_num_chunks": max_chunks}}


def dense(sq, sk, slices):
    from oracle import oracle

    qr = [s[0:2] for s in slices]
    kr = [s[2:4] for s in slices]
    ty = [s[4] for s in slices]
    return oracle.dense_allowed(sq, sk, qr, kr, ty) if slices else np.zeros((sq, sk), np.int32)


@pytest.mark.parametrize("stages", [None, 3, 4])
@pytest.mark.parametrize("idx", range(len(MASKS)))
def test_exec_plan_covers_each_rank_exactly(built_lib, idx, stages):
    from paper_2505_13211_b200.planner import Mask, Scenario

    mask, cp, chunk = MASKS[idx]
    xp = Scenario(scenario(mask, cp, chunk, stages=stages)).exec_plan()
    if stages is not None:  # the multi-stage schedule is really planned
        assert xp["num_stages_bwd"] >= 3, xp["num_stages_bwd"]
        assert max(len(st["recv"]) for r in xp["ranks"] for st in r["bwd_stages"]) >= 2
    m = Mask(mask)
    S = m.seqlen_q
    glob = dense(S, S, [[*q, *k, t] for q, k, t in m.slices])
    cs, L = xp["chunk_size"], xp["local_tokens"]
    owner_local = {}  # global token -> (rank, local index)
    for r in xp["ranks"]:
        for i, c in enumerate(r["chunks"]):
            for t in range(cs):
                owner_local[c * cs + t] = (r["rank"], i * cs + t)
    total = np.zeros_like(glob)
    for r in xp["ranks"]:
        q_glob = np.array([c * cs + t for c in r["chunks"] for t in range(cs)])
        # host stage: local KV == local rows
        h = dense(L, L, r["host_slices"])
        total[np.ix_(q_glob, q_glob)] += h
        for key in ("fwd_stages", "bwd_stages"):
            got = np.zeros_like(glob)
            got[np.ix_(q_glob, q_glob)] += h
            for st in r[key]:
                kmap = np.zeros(st["buf_tokens"], np.int64)
                for src, gs, ge, src_local, off in st["recv"]:
                    assert owner_local[gs] == (src, src_local)
                    kmap[off:off + (ge - gs)] = np.arange(gs, ge)
                d = dense(L, st["buf_tokens"], st["slices"])
                np.add.at(got, (q_glob[:, None], kmap[None, :]), d)
            # every pass reproduces this rank's rows of the global mask exactly
            np.testing.assert_array_equal(got[q_glob], glob[q_glob])
            if key == "fwd_stages":
                recv = sum(st["buf_tokens"] for st in r[key])
                plan = Scenario(scenario(mask, cp, chunk, stages=stages)).plan()
                src_recv = plan["transfer_cast"]["sources"][r["rank"]]["recv_tokens"]
                assert recv == src_recv  # zero redundancy: exactly the planned GroupCast volume


def _exchange_worker(rank, world, port, mask, chunk, q, stages=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_13211_b200.cp import _stage_layouts
        from paper_2505_13211_b200.planner import Scenario

        xp = Scenario(scenario(mask, world, chunk, stages=stages)).exec_plan()
        ok = stages is None or (xp["num_stages_fwd"] >= 2 and xp["num_stages_bwd"] >= 2)
        me = xp["ranks"][rank]
        cs = xp["chunk_size"]
        ids = torch.tensor([c * cs + t for c in me["chunks"] for t in range(cs)], dtype=torch.int64)
        for key in ("fwd_stages", "bwd_stages"):
            for j, st in enumerate(_stage_layouts(xp, rank, key)):
                send = torch.cat([ids[a:b] for a, b in st.send_ranges]) if st.send_ranges else \
                    torch.empty(0, dtype=torch.int64)
                recv = torch.empty(st.buf_tokens, dtype=torch.int64)
                dist.all_to_all_single(recv, send, st.recv_splits, st.send_splits)
                want = []
                mine = me[key][j] if j < len(me[key]) else {"recv": []}
                for src, gs, ge, _sl, _off in mine["recv"]:
                    want += list(range(gs, ge))
                ok &= recv.tolist() == want
                # GroupReduce: return one count per received token; hosts add them up
                back = torch.empty(sum(st.send_splits), dtype=torch.int64)
                dist.all_to_all_single(back, torch.ones(st.buf_tokens, dtype=torch.int64),
                                       st.send_splits, st.recv_splits)
                ok &= bool((back == 1).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stages", [None, 4])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_groupcast_groupreduce_exchange_gloo(built_lib, world, stages):
    """Every stage's all-to-all delivers exactly the planned receive buffer
    (and the transposed GroupReduce returns one partial per sent token),
    with one stage and with the multi-stage split (stages=4: 2-4 fwd, 4 bwd)."""
    mask = {"seqlen": 512, "pattern": "varlen_block_causal", "params": {"sample_lengths": [256, 256],
                                                                        "block_size": 32}}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world + (20 if stages else 0)
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, mask, 16, q, stages))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


@pytest.mark.parametrize("mask", [
    {"seqlen": 4096, "pattern": "causal"},
    {"seqlen": 8192, "pattern": "block_causal", "params": {"block_size": 1024}},
    {"seqlen": 4096, "pattern": "varlen_block_causal_last_global",
     "params": {"sample_lengths": [2048, 1024, 1024], "block_size": 512}},
])
@pytest.mark.parametrize("cp", [2, 4, 8])
def test_ring_plan_covers_mask(built_lib, mask, cp):
    """Ring-attention baseline work lists (zigzag chunks x source rank) cover
    the mask's MULTIPLICITY area exactly, and stay inside the local buffers."""
    from paper_2505_13211_b200.planner import debug_eval

    S = mask["seqlen"]
    cs = S // (2 * cp)
    areas = debug_eval("shard", mask=mask, chunk=cs)
    asg = debug_eval("zigzag", areas=areas, cp=cp)["assignment"]
    chunks = [[i for i, a in enumerate(asg) if a == r] for r in range(cp)]
    assert sorted(sum(chunks, [])) == list(range(2 * cp))
    total = 0
    for r in range(cp):
        for s in range(cp):
            sl = debug_eval("chunk_pair_slices", mask=mask, chunk=cs, q_chunks=chunks[r], k_chunks=chunks[s])
            for qs, qe, ks, ke, _t in sl:
                assert 0 <= qs < qe <= len(chunks[r]) * cs and 0 <= ks < ke <= len(chunks[s]) * cs
            total += sum(debug_eval("slice_area", slice=x) for x in sl)
    assert total == debug_eval("mask", mask=mask)["area_multiplicity"]


def _ulysses_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_13211_b200.ulysses import _heads_to_tokens, _tokens_to_heads

        S, H, d = 8 * world, 2 * world, 3
        # value = token * 1000 + head * 10 + lane, so every element names its place
        full = (torch.arange(S)[:, None, None] * 1000 + torch.arange(H)[None, :, None] * 10
                + torch.arange(d)[None, None, :]).to(torch.float32)
        L = S // world
        shard = full[rank * L:(rank + 1) * L].contiguous()
        hl = H // world
        heads = _tokens_to_heads(shard, world, None)
        ok = torch.equal(heads, full[:, rank * hl:(rank + 1) * hl])
        ok &= torch.equal(_heads_to_tokens(heads, world, None), shard)
        lse_full = full[:, :, 0].t().contiguous()  # [H, S]
        lse_h = lse_full[rank * hl:(rank + 1) * hl]  # this rank's heads, every token
        back = _heads_to_tokens(lse_h.t().contiguous(), world, None).t()
        ok &= torch.equal(back, lse_full[:, rank * L:(rank + 1) * L])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ulysses_all_to_all_layout_gloo(world):
    """Ulysses CP (ulysses.py): token shard -> head shard over the whole
    sequence and back, and the LSE [heads, tokens] exchange, on gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650 + world
    procs = [ctx.Process(target=_ulysses_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res
