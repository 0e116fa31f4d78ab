"""Ring-attention context-parallel baseline on the same FFA kernels
(the comparison of the paper's Figs. 32-33).

Dispatch is the reference's zigzag (dispatch.cpp:233-250, bit-exact through
the planner), every rank keeps its Q rows and passes its K/V block around
the ring: at step j rank r holds the K/V of rank (r - j) mod cp, computes
FFA(local Q, that block) restricted to the mask (slices from the planner's
region clipping, ``chunk_pair_slices``) and merges by LSE. The backward
sends each block's f32 dK/dV accumulator along with its K/V, so after cp
hops it is back at its owner. Unlike MagiAttention's GroupCast, every rank
receives every other rank's K/V whether or not its rows need it.

Transfers overlap compute: the K/V of step j+1 moves (NCCL send/recv on a
side stream) while step j computes; in the backward the dQ matmuls of step
j+1 run while the dK/dV accumulator of step j travels.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import _lib
from .ffa import FFAPlan
from .planner import debug_eval


class RingAttention:
    """Ring-attention CP over one mask; chunks_per_rank zigzag chunks per rank."""

    def __init__(self, mask: dict, num_heads_q: int, num_heads_k: int, head_dim: int,
                 chunks_per_rank: int = 2, group=None, device=None, softmax_scale: float | None = None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.hq, self.hk, self.d = num_heads_q, num_heads_k, head_dim
        self.scale = 1.0 / math.sqrt(head_dim) if softmax_scale is None else softmax_scale
        info = debug_eval("mask", mask=mask)
        S = int(info["json"]["seqlen_q"])
        n = chunks_per_rank * self.world
        if S % n:
            raise ValueError(f"seqlen {S} not divisible into {n} chunks")
        self.chunk_size = S // n
        areas = debug_eval("shard", mask=mask, chunk=self.chunk_size)
        asg = debug_eval("zigzag", areas=areas, cp=self.world)["assignment"]
        self.chunks_of = [[i for i, a in enumerate(asg) if a == r] for r in range(self.world)]
        self.chunks = self.chunks_of[self.rank]
        self.local_tokens = len(self.chunks) * self.chunk_size
        self.area_multiplicity = int(info["area_multiplicity"])
        self.plans: list[FFAPlan | None] = []
        L = self.local_tokens
        for src in range(self.world):
            sl = debug_eval("chunk_pair_slices", mask=mask, chunk=self.chunk_size, q_chunks=self.chunks,
                            k_chunks=self.chunks_of[src])
            self.plans.append(FFAPlan([s[0:2] for s in sl], [s[2:4] for s in sl], [s[4] for s in sl], L,
                                      len(self.chunks_of[src]) * self.chunk_size, head_dim) if sl else None)
        self.comm_stream = torch.cuda.Stream(self.device)
        # gloo point-to-point moves host memory only (the transport of ranks
        # that share a GPU): K/V are then staged through the host
        self.host_staged = dist.is_initialized() and dist.get_backend(group) != "nccl"
        self.L = _lib.lib()

    def local_token_index(self) -> torch.Tensor:
        cs = self.chunk_size
        return torch.cat([torch.arange(c * cs, (c + 1) * cs) for c in self.chunks])

    def _shift(self, tensors):
        """Send `tensors` to the next rank, receive same-shaped ones from the
        previous rank, on the comm stream. Returns (received, works)."""
        nxt, prv = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        if self.host_staged:
            with torch.cuda.stream(self.comm_stream):
                sends = [t.to("cpu") for t in tensors]
            recv_h = [torch.empty_like(t) for t in sends]
            ops = []
            for t, r in zip(sends, recv_h):
                ops.append(dist.P2POp(dist.isend, t, nxt, group=self.group))
                ops.append(dist.P2POp(dist.irecv, r, prv, group=self.group))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            with torch.cuda.stream(self.comm_stream):
                return [r.to(self.device) for r in recv_h], []
        with torch.cuda.stream(self.comm_stream):
            recv = [torch.empty_like(t) for t in tensors]
            ops = []
            for t, r in zip(tensors, recv):
                ops.append(dist.P2POp(dist.isend, t, nxt, group=self.group))
                ops.append(dist.P2POp(dist.irecv, r, prv, group=self.group))
            works = dist.batch_isend_irecv(ops)
        return recv, works

    def forward(self, q, k, v):
        from .ffa import ffa_forward

        L = self.local_tokens
        out = torch.zeros((L, self.hq, self.d), dtype=torch.float32, device=q.device)
        lse = torch.full((self.hq, L), -math.inf, dtype=torch.float32, device=q.device)
        cur = torch.cuda.current_stream(q.device)
        kc, vc = k, v
        for step in range(self.world):
            src = (self.rank - step) % self.world
            pending = None
            if step + 1 < self.world:
                self.comm_stream.wait_stream(cur)
                pending = self._shift([kc, vc])
            if self.plans[src] is not None:
                ffa_forward(self.plans[src], q, kc, vc, self.scale, out=out, lse=lse, accumulate=True)
            if pending is not None:
                (kn, vn), works = pending
                for w in works:
                    w.wait()
                cur.wait_stream(self.comm_stream)
                for t in (kc, vc):
                    t.record_stream(self.comm_stream)
                kc, vc = kn, vn
        out_bf = torch.empty((L, self.hq, self.d), dtype=torch.bfloat16, device=q.device)
        _lib.check(self.L.magiplan_cast_f32_bf16(out.data_ptr(), out_bf.data_ptr(), out.numel(), cur.cuda_stream))
        return out_bf, lse, out

    def backward(self, q, k, v, out_f32, lse, dout):
        L = self.local_tokens
        dev = q.device
        cur = torch.cuda.current_stream(dev)
        sp = cur.cuda_stream
        delta = torch.empty((self.hq, L), dtype=torch.float32, device=dev)
        _lib.check(self.L.magiplan_ffa_bwd_preprocess(out_f32.data_ptr(), dout.data_ptr(), delta.data_ptr(), L,
                                                      self.hq, self.d, _lib.F32, sp))
        dq = torch.zeros((L, self.hq, self.d), dtype=torch.float32, device=dev)
        kc, vc = k, v
        dkc = torch.zeros((L, self.hk, self.d), dtype=torch.float32, device=dev)
        dvc = torch.zeros_like(dkc)
        dkv_pending = None
        for step in range(self.world):
            src = (self.rank - step) % self.world
            kv_pending = None
            if step + 1 < self.world:
                self.comm_stream.wait_stream(cur)
                kv_pending = self._shift([kc, vc])
            plan = self.plans[src]
            if plan is not None:
                _lib.check(self.L.magiplan_ffa_bwd_dq(plan.handle, q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                                                      lse.data_ptr(), delta.data_ptr(), dout.data_ptr(),
                                                      dq.data_ptr(), self.hq, self.hk, self.scale, _lib.F32, 1, sp))
            if dkv_pending is not None:
                # this block's dK/dV accumulator, arriving from the previous rank
                (dkc, dvc), works = dkv_pending
                for w in works:
                    w.wait()
                cur.wait_stream(self.comm_stream)
            if plan is not None:
                _lib.check(self.L.magiplan_ffa_bwd_dkdv(plan.handle, q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                                                        lse.data_ptr(), delta.data_ptr(), dout.data_ptr(),
                                                        dkc.data_ptr(), dvc.data_ptr(), self.hq, self.hk,
                                                        self.scale, _lib.F32, 1, sp))
            if self.world > 1:
                self.comm_stream.wait_stream(cur)
                dkv_pending = self._shift([dkc, dvc])
                for t in (dkc, dvc):
                    t.record_stream(self.comm_stream)
            if kv_pending is not None:
                (kn, vn), works = kv_pending
                for w in works:
                    w.wait()
                cur.wait_stream(self.comm_stream)
                for t in (kc, vc):
                    t.record_stream(self.comm_stream)
                kc, vc = kn, vn
        if dkv_pending is not None:  # own block's accumulator, back home after cp hops
            (dkc, dvc), works = dkv_pending
            for w in works:
                w.wait()
            cur.wait_stream(self.comm_stream)
        outs = []
        for t in (dq, dkc, dvc):
            b = torch.empty(t.shape, dtype=torch.bfloat16, device=dev)
            _lib.check(self.L.magiplan_cast_f32_bf16(t.data_ptr(), b.data_ptr(), t.numel(), sp))
            outs.append(b)
        return tuple(outs)

    def flops(self) -> tuple[int, int]:
        fwd = 4 * self.area_multiplicity * self.hq * self.d
        return fwd, fwd * 5 // 2

    def comm_tokens(self) -> dict:
        """Tokens this rank receives per pass (K/V every step, dK/dV every step)."""
        kv = (self.world - 1) * self.local_tokens
        return {"fwd_cast_recv_tokens": kv, "bwd_cast_recv_tokens": kv,
                "bwd_reduce_recv_tokens": self.world * self.local_tokens if self.world > 1 else 0}
