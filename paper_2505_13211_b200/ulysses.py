"""Ulysses (all-to-all head-parallel) context-parallel mode on the same FFA
kernels (the second CP strategy; its schedule model is
the reference's ``simulate_ulysses``, sim.cpp:345-424).

Rank r owns the contiguous token shard [r*S/cp, (r+1)*S/cp) with every
head (the reference's ``local = seqlen / cp_size``, sim.cpp:385, and its
``seqlen % cp_size`` constraint, sim.cpp:375-381). One all-to-all turns
the shard into the whole sequence for heads [r*H/cp, (r+1)*H/cp); FFA runs
over the full mask on those heads; one all-to-all turns the output back.
GQA stays local to a rank: q-head group r maps onto kv-head group r, since
(hq/cp)/(hk/cp) = hq/hk. The backward mirrors it: dO goes head-sharded,
dQ/dK/dV come back token-sharded. Each all-to-all moves (cp-1)/cp of the
tensor, the ``moved`` volume the reference model charges (sim.cpp:355-372).
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import _lib
from .ffa import FFAPlan, ffa_backward, ffa_forward
from .planner import Mask


def _tokens_to_heads(x: torch.Tensor, world: int, group) -> torch.Tensor:
    """[L, H, ...] token shard, all heads -> [world*L, H/world, ...] all
    tokens, this rank's head group (token order = source-rank order)."""
    L, H = x.shape[0], x.shape[1]
    if world == 1:
        return x.contiguous()
    send = x.reshape(L, world, H // world, *x.shape[2:]).transpose(0, 1).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return recv.reshape(world * L, H // world, *x.shape[2:])


def _heads_to_tokens(x: torch.Tensor, world: int, group) -> torch.Tensor:
    """Inverse of _tokens_to_heads: [world*L, H/world, ...] -> [L, H, ...]."""
    S, Hl = x.shape[0], x.shape[1]
    if world == 1:
        return x.contiguous()
    L = S // world
    send = x.reshape(world, L, Hl, *x.shape[2:]).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return recv.transpose(0, 1).reshape(L, world * Hl, *x.shape[2:])


class UlyssesAttention:
    """Ulysses CP over one mask (dict spec or slice JSON, as ``Mask``)."""

    def __init__(self, mask: dict, num_heads_q: int, num_heads_k: int, head_dim: int, group=None,
                 device=None, softmax_scale: float | None = None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.hq, self.hk, self.d = num_heads_q, num_heads_k, head_dim
        self.scale = 1.0 / math.sqrt(head_dim) if softmax_scale is None else softmax_scale
        m = Mask(mask)
        S = m.seqlen_q
        if S % self.world:
            raise ValueError(f"constraint violated: seqlen % cp_size = 0 (seqlen {S}, cp_size {self.world})")
        if num_heads_q % self.world or num_heads_k % self.world:
            raise ValueError(f"Ulysses needs num_heads_q ({num_heads_q}) and num_heads_k ({num_heads_k}) "
                             f"divisible by cp_size ({self.world})")
        self.seqlen = S
        self.local_tokens = S // self.world
        self.area_multiplicity = m.area()
        sl = m.slices
        self.plan = FFAPlan([list(s[0]) for s in sl], [list(s[1]) for s in sl], [s[2] for s in sl], S,
                            m.seqlen_k, head_dim) if sl else None
        self.L = _lib.lib()

    def local_token_index(self) -> torch.Tensor:
        L = self.local_tokens
        return torch.arange(self.rank * L, (self.rank + 1) * L)

    def forward(self, q, k, v):
        """q [L, hq, d], k/v [L, hk, d] (this rank's token shard, bf16) ->
        (out bf16 [L, hq, d], lse [hq, L], out f32 [L, hq, d])."""
        w, g = self.world, self.group
        qh, kh, vh = (_tokens_to_heads(t, w, g) for t in (q, k, v))
        S, hl = self.seqlen, self.hq // w
        out_h = torch.zeros((S, hl, self.d), dtype=torch.float32, device=q.device)
        lse_h = torch.full((hl, S), -math.inf, dtype=torch.float32, device=q.device)
        if self.plan is not None:
            ffa_forward(self.plan, qh, kh, vh, self.scale, out=out_h, lse=lse_h)
        out32 = _heads_to_tokens(out_h, w, g)
        # lse [hl, S] -> token-major [S, hl] for the exchange, then back to [hq, L]
        lse = _heads_to_tokens(lse_h.t().contiguous(), w, g).t().contiguous()
        out = torch.empty((self.local_tokens, self.hq, self.d), dtype=torch.bfloat16, device=q.device)
        stream = torch.cuda.current_stream(q.device).cuda_stream
        _lib.check(self.L.magiplan_cast_f32_bf16(out32.data_ptr(), out.data_ptr(), out32.numel(), stream))
        # the head-sharded tensors are reused by the backward of THIS forward
        # only: keyed by the identity and version of every tensor involved
        self._saved = ((q, k, v, out32, lse), [t._version for t in (q, k, v, out32, lse)],
                       (qh, kh, vh, out_h, lse_h))
        return out, lse, out32

    def _matches(self, ts) -> bool:
        saved = getattr(self, "_saved", None)
        return (saved is not None and all(a is b for a, b in zip(saved[0], ts))
                and saved[1] == [t._version for t in ts])

    def backward(self, q, k, v, out_f32, lse, dout):
        """dQ, dK, dV (bf16, this rank's token shard). Reuses the head-sharded
        tensors of the forward that produced (out_f32, lse) when these are
        its outputs for the same q/k/v; otherwise (another forward ran in
        between, or different inputs) they are exchanged again from the
        arguments."""
        w, g = self.world, self.group
        if self._matches((q, k, v, out_f32, lse)):
            qh, kh, vh, out_h, lse_h = self._saved[2]
        else:
            qh, kh, vh, out_h = (_tokens_to_heads(t, w, g) for t in (q, k, v, out_f32))
            lse_h = _tokens_to_heads(lse.t().contiguous(), w, g).t().contiguous()
        doh = _tokens_to_heads(dout, w, g)
        if self.plan is None:
            dqh = torch.zeros(qh.shape, dtype=torch.float32, device=q.device)
            dkh = torch.zeros(kh.shape, dtype=torch.float32, device=q.device)
            dvh = torch.zeros_like(dkh)
        else:
            dqh, dkh, dvh = ffa_backward(self.plan, qh, kh, vh, out_h, lse_h, doh, self.scale,
                                         grad_dtype=torch.bfloat16)
        return tuple(_heads_to_tokens(t, w, g) for t in (dqh, dkh, dvh))

    def flops(self) -> tuple[int, int]:
        fwd = 4 * self.area_multiplicity * self.hq * self.d
        return fwd, fwd * 5 // 2

    def comm_tokens(self) -> dict:
        """Tokens (all heads) this rank receives per pass: q, k, v in and o out
        in the forward; dO in and dQ, dK, dV out in the backward."""
        moved = self.local_tokens * (self.world - 1) // self.world
        return {"fwd_a2a_tokens": 4 * moved, "bwd_a2a_tokens": 4 * moved}
