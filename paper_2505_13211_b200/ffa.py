"""Flexible Flash Attention (FFA) — torch-facing host API over the C ABI.

The operator surface mirrors MagiAttention's ``flex_flash_attn_func``
(§3.1: q/k ranges + per-slice attention type); the mask metadata
types are the reference planner's AttnSlice/AttnMask
(/root/reference/proj/include/magiplan/mask.hpp:59-99). Every call goes
through ``libmagiplan.so`` (``magiplan_ffa_*``); torch only provides device
memory and the current stream. There is no CPU or eager fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Sequence

import numpy as np
import torch

from . import _lib

SLICE_TYPES = {"full": 0, "causal": 1, "inv_causal": 2, "bi_causal": 3}


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class FFAPlan:
    """Device work list of one slice composition (magiplan_ffa_plan).

    Build once per mask and reuse across layers / steps / heads.
    """

    def __init__(self, q_ranges, k_ranges, types, seqlen_q: int, seqlen_k: int, head_dim: int):
        qr = np.ascontiguousarray(np.asarray(q_ranges, dtype=np.int64).reshape(-1, 2))
        kr = np.ascontiguousarray(np.asarray(k_ranges, dtype=np.int64).reshape(-1, 2))
        ty = np.asarray([SLICE_TYPES[t] if isinstance(t, str) else int(t) for t in
                         np.asarray(types, dtype=object).reshape(-1)], dtype=np.int32)
        if not (len(qr) == len(kr) == len(ty)):
            raise ValueError("q_ranges, k_ranges and types must have the same length")
        self.q_ranges, self.k_ranges, self.types = qr, kr, ty
        self.seqlen_q, self.seqlen_k, self.head_dim = int(seqlen_q), int(seqlen_k), int(head_dim)
        handle = C.c_void_p()
        L = _lib.lib()
        _lib.check(L.magiplan_ffa_plan_create(
            qr.ctypes.data_as(C.POINTER(C.c_int64)), kr.ctypes.data_as(C.POINTER(C.c_int64)),
            ty.ctypes.data_as(C.POINTER(C.c_int32)), len(ty), self.seqlen_q, self.seqlen_k,
            self.head_dim, C.byref(handle)))
        self._handle = handle

    @classmethod
    def from_mask(cls, mask, head_dim: int) -> "FFAPlan":
        sl = mask.slices
        return cls([s[0] for s in sl], [s[1] for s in sl], [s[2] for s in sl], mask.seqlen_q,
                   mask.seqlen_k, head_dim)

    @property
    def handle(self) -> C.c_void_p:
        return self._handle

    def describe(self) -> dict:
        import json

        out = C.c_void_p()
        _lib.check(_lib.lib().magiplan_ffa_plan_describe(self._handle, C.byref(out)))
        return json.loads(_lib.take_string(out))

    def prepare(self) -> None:
        """Upload the work lists to the current CUDA device now
        (magiplan_ffa_plan_prepare) instead of inside the first launch."""
        _lib.check(_lib.lib().magiplan_ffa_plan_prepare(self._handle))

    def area(self) -> int:
        return int(self.describe()["area_multiplicity"])

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().magiplan_ffa_plan_free(h)
            except Exception:
                pass


def _check_qkv(plan: FFAPlan, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous() or t.dim() != 3:
            raise ValueError(f"{name} must be a contiguous CUDA bf16 [tokens, heads, head_dim] tensor")
    if q.shape[0] != plan.seqlen_q or k.shape[0] != plan.seqlen_k or v.shape != k.shape:
        raise ValueError("q/k/v token counts do not match the plan")
    if q.shape[2] != plan.head_dim or k.shape[2] != plan.head_dim:
        raise ValueError("head_dim does not match the plan")


def _check_buf(name: str, t: torch.Tensor, shape: tuple, device: torch.device,
               dtypes: tuple = (torch.float32, torch.bfloat16)) -> None:
    """Caller-supplied output / auxiliary buffers are written through raw
    pointers: a wrong shape, dtype, device or layout is a ValueError here,
    never an out-of-bounds device write."""
    if not torch.is_tensor(t):
        raise ValueError(f"{name} must be a tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.dtype not in dtypes:
        raise ValueError(f"{name} must be one of {dtypes}, got {t.dtype}")
    if t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def ffa_forward(plan: FFAPlan, q, k, v, softmax_scale: float | None = None, *,
                out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                out_dtype: torch.dtype = torch.bfloat16, accumulate: bool = False):
    """O, LSE = FFA(q, k, v) over the plan's slices (magiplan_ffa_fwd).

    With ``accumulate=True`` (f32 ``out``) the call merges into an existing
    (out, lse) pair with the log-sum-exp correction — the per-stage merge of
    the context-parallel forward.
    """
    _check_qkv(plan, q, k, v)
    sq, hq, d = q.shape
    hk = k.shape[1]
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    if out is None:
        out = torch.empty((sq, hq, d), dtype=out_dtype, device=q.device)
    if lse is None:
        lse = torch.empty((hq, sq), dtype=torch.float32, device=q.device)
    _check_buf("out", out, (sq, hq, d), q.device)
    _check_buf("lse", lse, (hq, sq), q.device, (torch.float32,))
    dt = _lib.F32 if out.dtype == torch.float32 else _lib.BF16
    with torch.cuda.device(q.device):  # plan upload and launch on q's device
        _lib.check(_lib.lib().magiplan_ffa_fwd(
            plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr(),
            hq, hk, scale, dt, int(accumulate), _stream_ptr(q.device)))
    return out, lse


def ffa_backward(plan: FFAPlan, q, k, v, out, lse, dout, softmax_scale: float | None = None, *,
                 delta: torch.Tensor | None = None, dq=None, dk=None, dv=None,
                 grad_dtype: torch.dtype = torch.bfloat16, accumulate: bool = False):
    """dQ, dK, dV of FFA (magiplan_ffa_bwd_preprocess + magiplan_ffa_bwd)."""
    _check_qkv(plan, q, k, v)
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    dev = q.device
    stream = _stream_ptr(dev)
    L = _lib.lib()
    _check_buf("out", out, (sq, hq, d), dev)
    _check_buf("lse", lse, (hq, sq), dev, (torch.float32,))
    _check_buf("dout", dout, (sq, hq, d), dev, (torch.bfloat16,))
    with torch.cuda.device(dev):  # plan upload and launches on q's device
        if delta is None:
            delta = torch.empty((hq, sq), dtype=torch.float32, device=dev)
            _lib.check(L.magiplan_ffa_bwd_preprocess(
                out.data_ptr(), dout.data_ptr(), delta.data_ptr(), sq, hq, d,
                _lib.F32 if out.dtype == torch.float32 else _lib.BF16, stream))
        _check_buf("delta", delta, (hq, sq), dev, (torch.float32,))
        if dq is None:
            dq = torch.empty((sq, hq, d), dtype=grad_dtype, device=dev)
        if dk is None:
            dk = torch.empty((sk, hk, d), dtype=grad_dtype, device=dev)
        if dv is None:
            dv = torch.empty((sk, hk, d), dtype=grad_dtype, device=dev)
        _check_buf("dq", dq, (sq, hq, d), dev)
        _check_buf("dk", dk, (sk, hk, d), dev, (dq.dtype,))
        _check_buf("dv", dv, (sk, hk, d), dev, (dq.dtype,))
        gdt = _lib.F32 if dq.dtype == torch.float32 else _lib.BF16
        _lib.check(L.magiplan_ffa_bwd(
            plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), lse.data_ptr(), delta.data_ptr(),
            dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), hq, hk, scale, gdt,
            int(accumulate), stream))
    return dq, dk, dv


_PLAN_CACHE: dict = {}


def get_plan(q_ranges, k_ranges, types, seqlen_q, seqlen_k, head_dim,
             device: torch.device | None = None) -> FFAPlan:
    """Cached plan per (slice list, sizes, device): a plan's work lists live
    on the device of its first launch (magiplan_ffa_plan_prepare)."""
    qr = np.asarray(q_ranges.cpu() if torch.is_tensor(q_ranges) else q_ranges, dtype=np.int64)
    kr = np.asarray(k_ranges.cpu() if torch.is_tensor(k_ranges) else k_ranges, dtype=np.int64)
    if types is None:
        ty = np.zeros(len(qr.reshape(-1, 2)), dtype=np.int32)
    else:
        ty = np.asarray(types.cpu() if torch.is_tensor(types) else
                        [SLICE_TYPES[t] if isinstance(t, str) else int(t) for t in types], dtype=np.int32)
    key = (qr.tobytes(), kr.tobytes(), ty.tobytes(), int(seqlen_q), int(seqlen_k), int(head_dim),
           str(device))
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = FFAPlan(qr, kr, ty, seqlen_q, seqlen_k, head_dim)
        if len(_PLAN_CACHE) > 64:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = plan
    return plan


class _FlexFlashAttn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, plan, softmax_scale):
        out, lse = ffa_forward(plan, q, k, v, softmax_scale)
        ctx.save_for_backward(q, k, v, out, lse)
        ctx.plan, ctx.scale = plan, softmax_scale
        ctx.mark_non_differentiable(lse)
        return out, lse

    @staticmethod
    def backward(ctx, dout, _dlse):
        q, k, v, out, lse = ctx.saved_tensors
        dq, dk, dv = ffa_backward(ctx.plan, q, k, v, out, lse, dout.contiguous(), ctx.scale)
        return dq, dk, dv, None, None


def flex_flash_attn_func(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_ranges, k_ranges,
                         attn_type_map: Sequence[int] | torch.Tensor | None = None,
                         softmax_scale: float | None = None):
    """MagiAttention-style entry point: ``(out, lse)`` for the slice list.

    q: [sq, hq, d], k/v: [sk, hk, d] bf16 CUDA; q_ranges/k_ranges: [n, 2]
    half-open token ranges; attn_type_map: [n] of 0 full, 1 causal,
    2 inv_causal, 3 bi_causal (default all full). Differentiable w.r.t. q, k, v.
    """
    plan = get_plan(q_ranges, k_ranges, attn_type_map, q.shape[0], k.shape[0], q.shape[2], q.device)
    return _FlexFlashAttn.apply(q, k, v, plan, softmax_scale)
