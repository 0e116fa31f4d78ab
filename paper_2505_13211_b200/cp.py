"""Context-parallel FFA executor: dispatch + GroupCast / GroupReduce + staged
FFA with overlap, one process per GPU over torch.distributed (NCCL).

This is the real counterpart of the reference's ``simulate_magi`` schedule
(/root/reference/proj/src/sim.cpp:174-259): the plan (dispatch,
zero-redundant transfer tables, stage split) comes from the planner through
``magiplan_scenario_exec_plan``; every stage is executed with the sm_100a
FFA kernels; communication runs on its own CUDA streams.

Forward, per rank (§4.2, Alg. 2):
    step 0      FFA(local Q, local KV)                 || GroupCast(stage 1)
    step j      FFA(local Q, stage-j KV), LSE merge    || GroupCast(stage j+1)
Backward:
    step 0      dQ, dK, dV from local KV                || GroupCast(stage 1)
    step j      dQ += ..., partial dK/dV of stage j     || GroupCast(j+1) || GroupReduce(j-1)
    final       GroupReduce(last stage)
GroupCast = range-gather kernel + NCCL all_to_all_single (grouped by source
rank, which is the receive-buffer layout the planner emits). GroupReduce =
the transposed all-to-all of f32 partial dK/dV followed by the deterministic
range scatter-add kernel, one source rank at a time in rank order.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import _lib
from .ffa import FFAPlan
from .planner import Scenario


@dataclass
class StageLayout:
    """Communication + compute layout of one stage on one rank."""

    buf_tokens: int
    recv_splits: list[int]                 # tokens received from each source rank
    send_splits: list[int]                 # tokens sent to each destination rank
    send_ranges: list[tuple[int, int]]     # local [start, end) rows, send-buffer order
    send_by_dst: list[list[int]]           # indices into send_ranges per destination
    slices: list[list[int]]                # [qs, qe, ks, ke, type] local q / buffer k
    plan: FFAPlan | None = None
    dev: dict = field(default_factory=dict)


def _stage_layouts(xplan: dict, rank: int, key: str) -> list[StageLayout]:
    cp = xplan["cp_size"]
    ranks = xplan["ranks"]
    n = max(len(r[key]) for r in ranks)
    out = []
    for j in range(n):
        mine = ranks[rank][key][j] if j < len(ranks[rank][key]) else {"buf_tokens": 0, "recv": [], "slices": []}
        recv_splits = [0] * cp
        for src, gs, ge, _sl, _off in mine["recv"]:
            recv_splits[src] += ge - gs
        send_splits = [0] * cp
        send_ranges: list[tuple[int, int]] = []
        send_by_dst: list[list[int]] = [[] for _ in range(cp)]
        for dst in range(cp):
            st = ranks[dst][key][j] if j < len(ranks[dst][key]) else None
            if st is None:
                continue
            for src, gs, ge, src_local, _off in st["recv"]:
                if src != rank:
                    continue
                send_by_dst[dst].append(len(send_ranges))
                send_ranges.append((src_local, src_local + (ge - gs)))
                send_splits[dst] += ge - gs
        out.append(StageLayout(mine["buf_tokens"], recv_splits, send_splits, send_ranges,
                               send_by_dst, mine["slices"]))
    return out


def _new_group(ranks: list[int]):
    """A second NCCL communicator over the same ranks, on high-priority
    streams. Collective: every rank calls it in the same order."""
    opts = None
    if dist.get_backend() == "nccl":
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
    return dist.new_group(ranks=ranks, pg_options=opts)


def _ranges_tensor(ranges: list[tuple[int, int]], device) -> tuple[torch.Tensor, torch.Tensor]:
    r = torch.tensor(ranges if ranges else [[0, 0]], dtype=torch.int64).reshape(-1, 2)
    lens = (r[:, 1] - r[:, 0]).tolist() if ranges else [0]
    offs = [0]
    for x in lens[:-1]:
        offs.append(offs[-1] + x)
    return r.to(device), torch.tensor(offs, dtype=torch.int64, device=device)


class CPAttention:
    """Context-parallel FFA over one scenario (mask + dispatch + stages).

    Every rank builds the same executor plan from the same scenario (the
    planner is deterministic), then keeps only its own view.
    """

    def __init__(self, scenario: dict | str, num_heads_q: int, num_heads_k: int, head_dim: int,
                 group=None, device=None, softmax_scale: float | None = None, transport: str = "nccl"):
        """transport: "nccl" (GroupCast / GroupReduce as NCCL all-to-alls) or
        "p2p" (the forward GroupCast as one range-copy kernel writing straight
        into the consumers' receive buffers over NVLink, mapped with CUDA IPC,
        ordered by stream-side flags; one rank per GPU, GroupReduce on NCCL)."""
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport {transport!r}: 'nccl' or 'p2p'")
        self.transport = transport
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.hq, self.hk, self.d = num_heads_q, num_heads_k, head_dim
        self.scale = 1.0 / math.sqrt(head_dim) if softmax_scale is None else softmax_scale
        self.xplan = Scenario(scenario).exec_plan()
        if self.xplan["cp_size"] != self.world:
            raise ValueError(f"scenario cp_size {self.xplan['cp_size']} != world size {self.world}")
        me = self.xplan["ranks"][self.rank]
        self.chunks = me["chunks"]
        self.chunk_size = self.xplan["chunk_size"]
        self.local_tokens = self.xplan["local_tokens"]
        L = self.local_tokens
        hs = me["host_slices"]
        self.host_plan = FFAPlan([s[0:2] for s in hs], [s[2:4] for s in hs], [s[4] for s in hs], L, L,
                                 head_dim) if hs else None
        self.fwd_stages = _stage_layouts(self.xplan, self.rank, "fwd_stages")
        self.bwd_stages = _stage_layouts(self.xplan, self.rank, "bwd_stages")
        for st in self.fwd_stages + self.bwd_stages:
            if st.slices:
                st.plan = FFAPlan([s[0:2] for s in st.slices], [s[2:4] for s in st.slices],
                                  [s[4] for s in st.slices], L, st.buf_tokens, head_dim)
            st.dev["send"] = _ranges_tensor(st.send_ranges, self.device)
            per_dst = []
            for dst in range(self.world):
                rr = [st.send_ranges[i] for i in st.send_by_dst[dst]]
                per_dst.append(_ranges_tensor(rr, self.device) + (sum(b - a for a, b in rr),))
            st.dev["per_dst"] = per_dst
        # Work lists go to the device now (one synchronous upload per plan),
        # not inside the first step that launches them.
        for pl in [self.host_plan] + [st.plan for st in self.fwd_stages + self.bwd_stages]:
            if pl is not None:
                with torch.cuda.device(self.device):
                    pl.prepare()
        # High-priority streams: the block scheduler hands freed SMs to the
        # gather / scatter-add / NCCL kernels ahead of queued FFA CTAs, the
        # B200 counterpart of the paper's "communication kernel picked first"
        # (footnote 7).
        lo, hi = torch.cuda.Stream.priority_range()
        self.comm_stream = torch.cuda.Stream(self.device, priority=hi)
        self.reduce_stream = torch.cuda.Stream(self.device, priority=hi)
        self._probe_stream = torch.cuda.Stream(self.device)
        # GroupCast and GroupReduce on two communicators, so the all-to-alls
        # of cast(j+1) and reduce(j-1) run concurrently instead of queueing on
        # one NCCL stream (footnote 8).
        self.cast_group, self.reduce_group = self.group, self.group
        if self.world > 1:
            ranks = dist.get_process_group_ranks(group) if group is not None else list(range(self.world))
            self.cast_group = _new_group(ranks)
            self.reduce_group = _new_group(ranks)
        self.L = _lib.lib()
        self.timeline: list | None = None  # set to [] to record per-stage CUDA events
        self._p2p: list[dict] = []
        self._p2p_bwd: list[dict] = []
        self._p2p_epoch = 0
        self._p2p_bepoch = 0
        self._p2p_owned: list[int] = []
        self._p2p_opened: list[int] = []
        if transport == "p2p" and self.world > 1:
            self._setup_p2p()

    # ------------------------------------------------------------ peer memory
    def _setup_p2p(self):
        """Per stage of both passes: receive buffers and a flag block in
        IPC-exportable memory, handles exchanged once, the peers' buffers
        mapped, and the device arrays of the fused gather-and-send kernel
        built from the executor plan (every consumer's receive entries from
        this rank, at their buffer rows). Backward stages also get f32
        partial dK / dV buffers the owners read back for the GroupReduce.
        Flag block of a stage (uint32, index = peer rank): [ready | consumed
        | partials ready | partials read], each written by the peer into this
        rank's block."""
        import ctypes as C

        cp, me, L = self.world, self.rank, self.L
        if cp > 32:
            raise ValueError("p2p transport: at most 32 ranks (flag masks)")
        row = self.hk * self.d * 2

        def alloc(nbytes):
            ptr, h = C.c_void_p(), C.create_string_buffer(64)
            _lib.check(L.magiplan_p2p_malloc(nbytes, C.byref(ptr), h))
            self._p2p_owned.append(ptr.value)
            return ptr.value, h.raw

        def view(ptr, n, typestr, dtype):
            class _Raw:
                __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                            "version": 3, "strides": None}
            return torch.as_tensor(_Raw(), device=self.device).view(dtype)

        def dev64(vals):
            return torch.tensor(vals if vals else [0], dtype=torch.int64, device=self.device)

        ranks = self.xplan["ranks"]
        passes = (("fwd_stages", self.fwd_stages, False), ("bwd_stages", self.bwd_stages, True))
        local, handles = [], []
        for _key, stages, bwd in passes:
            for st in stages:
                n = max(st.buf_tokens, 1) * self.hk * self.d
                bufs = [alloc(n * 2), alloc(n * 2)]           # K, V receive buffers (bf16)
                if bwd:
                    bufs += [alloc(n * 4), alloc(n * 4)]      # partial dK, dV (f32)
                fp, fh = alloc(4 * cp * 4)
                view(fp, 4 * cp, "<i4", torch.int32).zero_()
                local.append(([b[0] for b in bufs], fp))
                handles.append(([b[1] for b in bufs], fh))
        torch.cuda.synchronize(self.device)
        every = [None] * cp
        dist.all_gather_object(every, handles, group=self.group)

        idx = 0
        for key, stages, bwd in passes:
            out = []
            for j, st in enumerate(stages):
                ptrs, fp = local[idx]
                peer = {}
                for d in range(cp):
                    if d == me:
                        continue
                    hb, hf = every[d][idx]
                    opened = []
                    for h in hb + [hf]:
                        o = C.c_void_p()
                        _lib.check(L.magiplan_p2p_open(h, C.byref(o)))
                        self._p2p_opened.append(o.value)
                        opened.append(o.value)
                    peer[d] = opened          # [k, v, (dk, dv,) flags]
                idx += 1
                ranges, offs, kbase, vbase, drow, acc = [], [], [], [], [], 0
                dests, per_dst = [], {}
                for d in range(cp):
                    if d == me or j >= len(ranks[d][key]):
                        continue
                    mine = [e for e in ranks[d][key][j]["recv"] if e[0] == me]
                    if not mine:
                        continue
                    dests.append(d)
                    rr, ro, rb_dk, rb_dv, rrow, racc = [], [], [], [], [], 0
                    for _src, gs, ge, src_local, buf_off in mine:
                        ranges += [src_local, src_local + (ge - gs)]
                        offs.append(acc)
                        acc += ge - gs
                        kbase.append(peer[d][0])
                        vbase.append(peer[d][1])
                        drow.append(buf_off)
                        if bwd:
                            rr += [src_local, src_local + (ge - gs)]
                            ro.append(racc)
                            racc += ge - gs
                            rb_dk.append(peer[d][2])
                            rb_dv.append(peer[d][3])
                            rrow.append(buf_off)
                    if bwd:
                        per_dst[d] = (dev64(rr), dev64(ro), dev64(rb_dk), dev64(rb_dv), dev64(rrow),
                                      len(ro), racc)
                srcs = sorted({e[0] for e in ranks[me][key][j]["recv"]}) if j < len(ranks[me][key]) else []
                nt = max(st.buf_tokens, 1) * self.hk * self.d
                P = {
                    "kb": view(ptrs[0], nt, "<i2", torch.bfloat16).view(-1, self.hk, self.d)[:st.buf_tokens],
                    "vb": view(ptrs[1], nt, "<i2", torch.bfloat16).view(-1, self.hk, self.d)[:st.buf_tokens],
                    "flags": fp, "rows": acc, "n": len(offs), "row_bytes": row,
                    "ranges": dev64(ranges), "offs": dev64(offs), "drow": dev64(drow),
                    "kbase": dev64(kbase), "vbase": dev64(vbase),
                    # cast: producer raises consumers' ready[me], waits its own consumed[d]
                    "sig_send": dev64([peer[d][-1] + 4 * me for d in dests]), "n_dest": len(dests),
                    "mask_dest": sum(1 << d for d in dests),
                    "sig_recv": dev64([peer[s_][-1] + 4 * (cp + me) for s_ in srcs]), "n_src": len(srcs),
                    "mask_src": sum(1 << s_ for s_ in srcs),
                }
                if bwd:
                    P["dkb"] = view(ptrs[2], nt, "<f4", torch.float32).view(-1, self.hk, self.d)[:st.buf_tokens]
                    P["dvb"] = view(ptrs[3], nt, "<f4", torch.float32).view(-1, self.hk, self.d)[:st.buf_tokens]
                    # reduce: consumer raises owners' pready[me]; owner raises consumers' pdone[me]
                    P["sig_pready"] = dev64([peer[s_][-1] + 4 * (2 * cp + me) for s_ in srcs])
                    P["sig_pdone"] = dev64([peer[d][-1] + 4 * (3 * cp + me) for d in dests])
                    P["per_dst"] = per_dst
                out.append(P)
            if bwd:
                self._p2p_bwd = out
            else:
                self._p2p = out

    def _flags_wait(self, P, block: int, mask: int, value: int, stream):
        _lib.check(self.L.magiplan_flags_wait(P["flags"] + 4 * block * self.world, mask, value, stream.cuda_stream))

    def _flags_signal(self, ptrs, n: int, value: int, stream):
        _lib.check(self.L.magiplan_flags_signal(ptrs.data_ptr(), n, value, stream.cuda_stream))

    def close(self):
        """Release the peer-memory mappings and buffers (p2p transport).
        Safe once this rank's passes have completed: a backward pass ends only
        after the owners have read its partials, and peers write into this
        rank's receive buffers only inside passes it takes part in."""
        if not self._p2p_owned and not self._p2p_opened:
            return
        torch.cuda.synchronize(self.device)
        for ptr in self._p2p_opened:
            self.L.magiplan_p2p_close(ptr)
        for ptr in self._p2p_owned:
            self.L.magiplan_p2p_free(ptr)
        self._p2p_opened, self._p2p_owned, self._p2p, self._p2p_bwd = [], [], [], []

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown / CUDA already torn down
            pass

    def _cast_p2p(self, P: dict, epoch: int, k: torch.Tensor, v: torch.Tensor):
        """GroupCast of one stage over peer memory, on the comm stream: wait
        until every consumer has released this stage's buffer from the
        previous pass, copy the ranges into the consumers' buffers, then
        raise their ready flags. Same return shape as _cast."""
        L = self.L
        sp = self.comm_stream.cuda_stream
        with torch.cuda.stream(self.comm_stream):
            e0 = self._ev(self.comm_stream)
            self._flags_wait(P, 1, P["mask_dest"], epoch - 1, self.comm_stream)
            if P["n"]:
                for src, base in ((k, P["kbase"]), (v, P["vbase"])):
                    _lib.check(L.magiplan_range_copy_to(src.data_ptr(), P["ranges"].data_ptr(),
                                                        P["offs"].data_ptr(), base.data_ptr(), P["drow"].data_ptr(),
                                                        P["n"], P["rows"], P["row_bytes"], sp))
            self._flags_signal(P["sig_send"], P["n_dest"], epoch, self.comm_stream)
        return P["kb"], P["vb"], [], None, e0

    def _reduce_p2p(self, P: dict, epoch: int, dk, dv):
        """GroupReduce of one backward stage over peer memory, on the reduce
        stream: wait for the consumers' partials, then per consumer in rank
        order add its partial dK / dV rows (read over NVLink) into this
        rank's dK / dV, then tell it the buffers may be reused."""
        rs = self.reduce_stream
        self._flags_wait(P, 2, P["mask_dest"], epoch, rs)
        row_elems = self.hk * self.d
        for d in sorted(P["per_dst"]):
            rr, ro, bdk, bdv, rrow, n, rows = P["per_dst"][d]
            for acc, base in ((dk, bdk), (dv, bdv)):
                _lib.check(self.L.magiplan_range_scatter_add_from(
                    acc.data_ptr(), rr.data_ptr(), ro.data_ptr(), base.data_ptr(), rrow.data_ptr(), n, rows,
                    row_elems, rs.cuda_stream))
        self._flags_signal(P["sig_pdone"], P["n_dest"], epoch, rs)

    # ------------------------------------------------------------ tracing
    def _ev(self, stream):
        if self.timeline is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def _span(self, pass_, task, j, e0, e1):
        if self.timeline is not None:
            self.timeline.append((pass_, task, j, e0, e1))

    def timeline_ms(self, origin: "torch.cuda.Event") -> list[dict]:
        """Recorded spans in ms relative to `origin` (after a synchronize)."""
        out = []
        for pass_, task, j, e0, e1 in self.timeline or []:
            out.append({"pass": pass_, "task": task, "stage": j,
                        "start_ms": origin.elapsed_time(e0), "end_ms": origin.elapsed_time(e1)})
        return out

    # ------------------------------------------------------------ data layout
    def local_token_index(self) -> torch.Tensor:
        """Global token ids of this rank's local rows (chunk order)."""
        cs = self.chunk_size
        idx = [torch.arange(c * cs, (c + 1) * cs) for c in self.chunks]
        return torch.cat(idx) if idx else torch.empty(0, dtype=torch.int64)

    # ------------------------------------------------------------ primitives
    def _gather(self, src: torch.Tensor, st: StageLayout, stream) -> torch.Tensor:
        rows = sum(st.send_splits)
        out = torch.empty((rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        if rows:
            ranges, offs = st.dev["send"]
            row_bytes = src[0].numel() * src.element_size()
            _lib.check(self.L.magiplan_range_gather(src.data_ptr(), out.data_ptr(), ranges.data_ptr(),
                                                    offs.data_ptr(), len(st.send_ranges), rows,
                                                    row_bytes, stream.cuda_stream))
        return out

    def _cast(self, st: StageLayout, k: torch.Tensor, v: torch.Tensor):
        """GroupCast of stage `st`: range gather on the comm stream, then the
        all-to-all on the cast communicator. Returns (k_buf, v_buf, works,
        send buffers, start event). The send buffers must outlive the works:
        callers keep them until the compute stream has waited on every work
        of the pass (so reuse by a later gather on the comm stream, which
        first waits on the compute stream, is ordered after the NCCL read)."""
        with torch.cuda.stream(self.comm_stream):
            e0 = self._ev(self.comm_stream)
            ks = self._gather(k, st, self.comm_stream)
            vs = self._gather(v, st, self.comm_stream)
            kb = torch.empty((st.buf_tokens, self.hk, self.d), dtype=k.dtype, device=k.device)
            vb = torch.empty_like(kb)
            works = []
            if self.world > 1:
                works.append(dist.all_to_all_single(kb, ks, st.recv_splits, st.send_splits,
                                                    group=self.cast_group, async_op=True))
                works.append(dist.all_to_all_single(vb, vs, st.recv_splits, st.send_splits,
                                                    group=self.cast_group, async_op=True))
        return kb, vb, works, (ks, vs), e0

    def _cast_done(self, pass_, j, works, e0):
        """Make the compute stream wait for a GroupCast; trace its end."""
        cur = torch.cuda.current_stream(self.device)
        if self.timeline is not None:
            with torch.cuda.stream(self._probe_stream):
                self._probe_stream.wait_stream(self.comm_stream)
                for w in works:
                    w.wait()
                self._span(pass_, "cast", j, e0, self._ev(self._probe_stream))
        for w in works:
            w.wait()
        cur.wait_stream(self.comm_stream)

    def _reduce(self, st: StageLayout, dk_buf, dv_buf, dk, dv):
        """GroupReduce of a stage's f32 partial dK/dV into the hosts' dK/dV:
        the transposed all-to-all on the reduce communicator (asynchronous;
        the reduce stream waits on it), then one scatter-add per source rank
        in rank order (deterministic sums). Returns the receive buffers,
        which the caller keeps alive until the pass ends."""
        with torch.cuda.stream(self.reduce_stream):
            rows = sum(st.send_splits)
            rk = torch.empty((rows, self.hk, self.d), dtype=torch.float32, device=dk.device)
            rv = torch.empty_like(rk)
            if self.world > 1:
                works = [dist.all_to_all_single(rk, dk_buf, st.send_splits, st.recv_splits,
                                                group=self.reduce_group, async_op=True),
                         dist.all_to_all_single(rv, dv_buf, st.send_splits, st.recv_splits,
                                                group=self.reduce_group, async_op=True)]
                for w in works:
                    w.wait()
            base = 0
            row_elems = self.hk * self.d
            sp = self.reduce_stream.cuda_stream
            for dst in range(self.world):  # fixed source-rank order => deterministic sums
                ranges, offs, n = st.dev["per_dst"][dst]
                if n:
                    for part, acc in ((rk, dk), (rv, dv)):
                        _lib.check(self.L.magiplan_range_scatter_add_f32(
                            part[base:].data_ptr(), acc.data_ptr(), ranges.data_ptr(), offs.data_ptr(),
                            len(st.send_by_dst[dst]), n, row_elems, sp))
                base += n
        return rk, rv

    # ------------------------------------------------------------ forward
    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
        """q: [L, hq, d], k/v: [L, hk, d] bf16 local shards (chunk order).
        Returns (out bf16 [L, hq, d], lse f32 [hq, L], out f32 for backward)."""
        from .ffa import ffa_forward

        L = self.local_tokens
        out = torch.empty((L, self.hq, self.d), dtype=torch.float32, device=q.device)
        lse = torch.empty((self.hq, L), dtype=torch.float32, device=q.device)
        cur = torch.cuda.current_stream(q.device)
        self.comm_stream.wait_stream(cur)
        keep = []  # receive and send buffers of every stage, until the pass ends
        p2p = bool(self._p2p)
        if p2p:
            self._p2p_epoch += 1
        cast = ((lambda j: self._cast_p2p(self._p2p[j], self._p2p_epoch, k, v)) if p2p
                else (lambda j: self._cast(self.fwd_stages[j], k, v)))
        # step 0: cast(1) is issued first, then the host-local FFA
        pending = cast(0) if self.fwd_stages else None
        e0 = self._ev(cur)
        if self.host_plan is not None:
            ffa_forward(self.host_plan, q, k, v, self.scale, out=out, lse=lse)
        else:
            out.zero_()
            lse.fill_(-math.inf)
        self._span("fwd", "ffa", 0, e0, self._ev(cur))
        for j, st in enumerate(self.fwd_stages):
            kb, vb, works, sent, ec = pending
            if not p2p:
                keep.append((kb, vb, sent))
            # step j+1: cast(j+2) || ffa(j+1)
            if j + 1 < len(self.fwd_stages):
                pending = cast(j + 1)
            if p2p:
                # the peers' copies into this rank's buffer have landed
                P = self._p2p[j]
                self._flags_wait(P, 0, P["mask_src"], self._p2p_epoch, cur)
                if self.timeline is not None:
                    self._span("fwd", "cast", j + 1, ec, self._ev(cur))
            else:
                self._cast_done("fwd", j + 1, works, ec)
            e0 = self._ev(cur)
            if st.plan is not None:
                ffa_forward(st.plan, q, kb, vb, self.scale, out=out, lse=lse, accumulate=True)
            self._span("fwd", "ffa", j + 1, e0, self._ev(cur))
            if p2p:
                # release the buffer: the producers may overwrite it next pass
                self._flags_signal(P["sig_recv"], P["n_src"], self._p2p_epoch, cur)
        out_bf = torch.empty((L, self.hq, self.d), dtype=torch.bfloat16, device=q.device)
        _lib.check(self.L.magiplan_cast_f32_bf16(out.data_ptr(), out_bf.data_ptr(), out.numel(),
                                                 cur.cuda_stream))
        for kb, vb, (ks, vs) in keep:  # stream-ordered frees after the compute stream's last use
            for t in (kb, vb):
                t.record_stream(cur)
        return out_bf, lse, out

    # ------------------------------------------------------------ backward
    def backward(self, q, k, v, out_f32, lse, dout):
        """Returns (dq, dk, dv) bf16 local shards."""
        L = self.local_tokens
        dev = q.device
        cur = torch.cuda.current_stream(dev)
        sp = cur.cuda_stream
        Ld = self.L
        delta = torch.empty((self.hq, L), dtype=torch.float32, device=dev)
        dq = torch.empty((L, self.hq, self.d), dtype=torch.float32, device=dev)
        dk = torch.empty((L, self.hk, self.d), dtype=torch.float32, device=dev)
        dv = torch.empty_like(dk)
        self.comm_stream.wait_stream(cur)
        keep = []
        p2p = bool(self._p2p_bwd)
        if p2p:
            self._p2p_bepoch += 1
        eb = self._p2p_bepoch
        cast = ((lambda j: self._cast_p2p(self._p2p_bwd[j], eb, k, v)) if p2p
                else (lambda j: self._cast(self.bwd_stages[j], k, v)))
        # step 0: cast(1) first, then preprocess + host-local dQ / dK / dV
        pending = cast(0) if self.bwd_stages else None
        e0 = self._ev(cur)
        _lib.check(Ld.magiplan_ffa_bwd_preprocess(out_f32.data_ptr(), dout.data_ptr(),
                                                  delta.data_ptr(), L, self.hq, self.d, _lib.F32, sp))
        if self.host_plan is not None:
            _lib.check(Ld.magiplan_ffa_bwd(self.host_plan.handle, q.data_ptr(), k.data_ptr(),
                                           v.data_ptr(), lse.data_ptr(), delta.data_ptr(),
                                           dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                           self.hq, self.hk, self.scale, _lib.F32, 0, sp))
        else:
            dq.zero_()
            dk.zero_()
            dv.zero_()
        self._span("bwd", "ffa", 0, e0, self._ev(cur))
        for j, st in enumerate(self.bwd_stages):
            kb, vb, works, sent, ec = pending
            # step j+1: cast(j+2) || ffa(j+1) || reduce(j), the reduce having
            # been issued on its own stream right after ffa(j)
            if j + 1 < len(self.bwd_stages):
                pending = cast(j + 1)
            if p2p:
                P = self._p2p_bwd[j]
                # the peers' K / V for this stage have landed, and the owners
                # have read last pass's partials out of dkb / dvb
                self._flags_wait(P, 0, P["mask_src"], eb, cur)
                self._flags_wait(P, 3, P["mask_src"], eb - 1, cur)
                dkb, dvb = P["dkb"], P["dvb"]
            else:
                self._cast_done("bwd", j + 1, works, ec)
                # the dK/dV pass writes every row of its partial buffers (keys no
                # slice reaches get zeros), so they need no initialisation
                dkb = torch.empty((st.buf_tokens, self.hk, self.d), dtype=torch.float32, device=dev)
                dvb = torch.empty_like(dkb)
            e0 = self._ev(cur)
            if st.plan is not None:
                # fresh partial dK/dV of the received keys; dQ added into the
                # running dQ of the earlier stages
                _lib.check(Ld.magiplan_ffa_bwd_stage(st.plan.handle, q.data_ptr(), kb.data_ptr(),
                                                     vb.data_ptr(), lse.data_ptr(), delta.data_ptr(),
                                                     dout.data_ptr(), dq.data_ptr(), dkb.data_ptr(),
                                                     dvb.data_ptr(), self.hq, self.hk, self.scale, sp))
            else:
                dkb.zero_()
                dvb.zero_()
            self._span("bwd", "ffa", j + 1, e0, self._ev(cur))
            if p2p:
                # release this stage's K / V buffer, publish the partials
                self._flags_signal(P["sig_recv"], P["n_src"], eb, cur)
                self._flags_signal(P["sig_pready"], P["n_src"], eb, cur)
            self.reduce_stream.wait_stream(cur)  # partial dK/dV of this stage (and dk/dv) ready
            er = self._ev(self.reduce_stream)
            if p2p:
                self._reduce_p2p(P, eb, dk, dv)
                recv = None
            else:
                recv = self._reduce(st, dkb, dvb, dk, dv)
            self._span("bwd", "reduce", j + 1, er, self._ev(self.reduce_stream))
            if not p2p:
                keep.append((kb, vb, sent, dkb, dvb, recv))
        cur.wait_stream(self.reduce_stream)
        if p2p:
            # the owners have read this pass's partials out of this rank's
            # buffers: once the pass completes, no peer touches them (so the
            # buffers may be freed after a stream synchronize)
            for P in self._p2p_bwd:
                self._flags_wait(P, 3, P["mask_src"], eb, cur)
        outs = []
        for t in (dq, dk, dv):
            b = torch.empty(t.shape, dtype=torch.bfloat16, device=dev)
            _lib.check(self.L.magiplan_cast_f32_bf16(t.data_ptr(), b.data_ptr(), t.numel(), sp))
            outs.append(b)
        # buffers allocated on the comm / reduce streams are freed here, after
        # the compute stream has waited on every NCCL work that touched them
        del keep
        return tuple(outs)

    # ------------------------------------------------------------ accounting
    def flops(self) -> tuple[int, int]:
        """Whole-job mask-aware FLOPs (fwd, bwd), reference sim.cpp:29-34."""
        fwd = 4 * int(self.xplan["area_multiplicity"]) * self.hq * self.d
        return fwd, fwd * 5 // 2

    def comm_tokens(self) -> dict:
        cast = sum(sum(st.recv_splits) for st in self.fwd_stages)
        return {"fwd_cast_recv_tokens": cast,
                "bwd_cast_recv_tokens": sum(sum(st.recv_splits) for st in self.bwd_stages),
                "bwd_reduce_recv_tokens": sum(sum(st.send_splits) for st in self.bwd_stages)}


class CPExecutorC:
    """The same schedule through the C ABI's own executor (magiplan_cp_*,
    csrc/host/cp_exec.cpp): what a C / C++ consumer of libmagiplan.so runs.
    Torch only provides device memory, the stream and the NCCL unique-id
    broadcast; the executor creates its own NCCL communicators."""

    def __init__(self, scenario: dict | str, num_heads_q: int, num_heads_k: int, head_dim: int,
                 group=None, device=None, softmax_scale: float | None = None, transport: str = "nccl"):
        import ctypes as C

        if transport not in ("nccl", "p2p"):
            raise ValueError(f"transport {transport!r}: 'nccl' or 'p2p'")

        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.hq, self.hk, self.d = num_heads_q, num_heads_k, head_dim
        self.scale = 1.0 / math.sqrt(head_dim) if softmax_scale is None else softmax_scale
        self.L = _lib.lib()
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(self.L.magiplan_cp_unique_id(uid))
        obj = [bytes(uid.raw)]
        if self.world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        uid = C.create_string_buffer(obj[0], 128)
        self._scen = Scenario(scenario)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.L.magiplan_cp_create_ex(self._scen._h, self.rank, uid, num_heads_q, num_heads_k,
                                                    head_dim, self.scale, 0 if transport == "nccl" else 1,
                                                    C.byref(h)))
        self._h = h
        out = C.c_void_p()
        _lib.check(self.L.magiplan_cp_describe(self._h, C.byref(out)))
        info = json.loads(_lib.take_string(out))
        self.chunks, self.chunk_size = info["chunks"], info["chunk_size"]
        self.local_tokens = info["local_tokens"]
        self.transport = info["transport"]
        self.xplan = {"num_stages_fwd": info["num_stages_fwd"], "num_stages_bwd": info["num_stages_bwd"],
                      "area_multiplicity": info["area_multiplicity"], "seqlen": self.local_tokens * self.world}

    def local_token_index(self) -> torch.Tensor:
        cs = self.chunk_size
        idx = [torch.arange(c * cs, (c + 1) * cs) for c in self.chunks]
        return torch.cat(idx) if idx else torch.empty(0, dtype=torch.int64)

    def forward(self, q, k, v):
        L = self.local_tokens
        out32 = torch.empty((L, self.hq, self.d), dtype=torch.float32, device=q.device)
        lse = torch.empty((self.hq, L), dtype=torch.float32, device=q.device)
        out = torch.empty((L, self.hq, self.d), dtype=torch.bfloat16, device=q.device)
        _lib.check(self.L.magiplan_cp_forward(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out32.data_ptr(),
                                              lse.data_ptr(), out.data_ptr(),
                                              torch.cuda.current_stream(q.device).cuda_stream))
        return out, lse, out32

    def backward(self, q, k, v, out_f32, lse, dout):
        dq = torch.empty_like(q)
        dk, dv = torch.empty_like(k), torch.empty_like(v)
        _lib.check(self.L.magiplan_cp_backward(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out_f32.data_ptr(),
                                               lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                                               dv.data_ptr(), torch.cuda.current_stream(q.device).cuda_stream))
        return dq, dk, dv

    def flops(self) -> tuple[int, int]:
        fwd = 4 * int(self.xplan["area_multiplicity"]) * self.hq * self.d
        return fwd, fwd * 5 // 2

    def comm_tokens(self) -> dict:
        return {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                torch.cuda.synchronize(self.device)
                self.L.magiplan_cp_free(h)
            except Exception:  # noqa: BLE001
                pass
