"""Independent fp32 reference of FFA at sizes the CPU oracle cannot finish,
computed densely with PyTorch on the GPU from the same bf16 inputs
(test infrastructure; nothing here is on the product path).

Mask semantics are the reference's: a slice allows row q the key columns
[lo, hi) of AttnSlice::row_cols (/root/reference/proj/src/mask.cpp:74-84),
and a (q, k) pair covered by m slices counts m times (MULTIPLICITY, the
kernel's semantics, mask.hpp:85). The weight matrix W[q, k] = number of
slices allowing (q, k) carries the multiplicity exactly:
    LSE_q = log sum_k W[q,k] exp(s_qk),  P = W exp(s - LSE),  O = P V,
    dS = P (dP - delta), dQ = scale dS K, dK = scale dS^T Q, dV = P^T dO.
Every quantity (LSE and delta included) is recomputed here from Q/K/V/dO;
nothing is taken from the kernel under test.
"""
from __future__ import annotations

import torch

FULL, CAUSAL, INV, BI = 0, 1, 2, 3


def _bounds(sl, rows: torch.Tensor):
    """Allowed [lo, hi) per row for one slice (empty outside its rows)."""
    (qs, qe), (ks, ke), t = sl
    lo = torch.full_like(rows, ks)
    hi = torch.full_like(rows, ke)
    if t in (INV, BI):
        lo = torch.clamp(ks + (rows - qs), max=ke)
    if t in (CAUSAL, BI):
        hi = torch.clamp(rows + ke - qe + 1, min=ks, max=ke)
    inside = (rows >= qs) & (rows < qe)
    return torch.where(inside, lo, 0), torch.where(inside, hi, 0)


def weights(slices, rows: torch.Tensor, cols: torch.Tensor) -> torch.Tensor:
    """W[len(rows), len(cols)] float32 multiplicity weights."""
    w = torch.zeros(len(rows), len(cols), dtype=torch.float32, device=rows.device)
    for sl in slices:
        lo, hi = _bounds(sl, rows)
        w += ((cols[None, :] >= lo[:, None]) & (cols[None, :] < hi[:, None])).float()
    return w


def _expand(x: torch.Tensor, grp: int) -> torch.Tensor:
    return x.repeat_interleave(grp, dim=1) if grp > 1 else x


def forward_all(q, k, v, slices, scale, rows_per_chunk: int = 512):
    """fp32 O [sq, hq, d] and LSE [hq, sq] for every row (chunked)."""
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    grp = hq // hk
    kf, vf = _expand(k.float(), grp), _expand(v.float(), grp)  # [sk, hq, d]
    cols = torch.arange(sk, device=q.device)
    out = torch.zeros(sq, hq, d, dtype=torch.float32, device=q.device)
    lse = torch.full((hq, sq), float("-inf"), dtype=torch.float32, device=q.device)
    for r0 in range(0, sq, rows_per_chunk):
        rows = torch.arange(r0, min(sq, r0 + rows_per_chunk), device=q.device)
        w = weights(slices, rows, cols)  # [n, sk]
        nz = (w > 0).any(0).nonzero().flatten()
        if nz.numel() == 0:
            continue
        c0, c1 = int(nz[0]), int(nz[-1]) + 1
        w = w[:, c0:c1]
        s = torch.einsum("nhd,khd->hnk", q[rows].float(), kf[c0:c1]) * scale  # [hq, n, kk]
        s = s.masked_fill(w[None] == 0, float("-inf"))
        m = s.amax(-1, keepdim=True).clamp_min(-1e30)
        e = torch.exp(s - m) * w[None]
        tot = e.sum(-1, keepdim=True)
        l = (m + torch.log(tot)).squeeze(-1)  # [hq, n]
        p = e / tot.clamp_min(1e-30)
        out[rows] = torch.einsum("hnk,khd->nhd", p, vf[c0:c1])
        lse[:, rows] = torch.where(tot.squeeze(-1) > 0, l, torch.full_like(l, float("-inf")))
    return out, lse


def rows_ref(q, k, v, do, slices, scale, rows: list[int], lse_all, out_all):
    """fp32 (O, LSE, dQ) of the given query rows; delta from the reference O."""
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    grp = hq // hk
    dev = q.device
    r = torch.tensor(rows, device=dev)
    cols = torch.arange(sk, device=dev)
    w = weights(slices, r, cols)
    kf, vf = _expand(k.float(), grp), _expand(v.float(), grp)
    s = torch.einsum("nhd,khd->hnk", q[r].float(), kf) * scale
    lse = lse_all[:, r]  # [hq, n]
    p = torch.exp(s - torch.where(torch.isfinite(lse), lse, 0)[..., None]) * w[None]
    dp = torch.einsum("nhd,khd->hnk", do[r].float(), vf)
    delta = (do[r].float() * out_all[r]).sum(-1).T  # [hq, n]
    ds = p * (dp - delta[..., None])
    dq = torch.einsum("hnk,khd->nhd", ds, kf) * scale
    return out_all[r], lse, dq


def keys_ref(q, k, v, do, slices, scale, keys: list[int], lse_all, out_all,
             rows_per_chunk: int = 2048):
    """fp32 (dK, dV) [len(keys), hk, d] of the given key rows, summed over
    every (row, slice) that reaches them and over the GQA group."""
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    grp = hq // hk
    dev = q.device
    c = torch.tensor(keys, device=dev)
    kf, vf = _expand(k[c].float(), grp), _expand(v[c].float(), grp)  # [m, hq, d]
    dk = torch.zeros(len(keys), hq, d, dtype=torch.float32, device=dev)
    dv = torch.zeros_like(dk)
    delta_all = (do.float() * out_all).sum(-1)  # [sq, hq]
    for r0 in range(0, sq, rows_per_chunk):
        rows = torch.arange(r0, min(sq, r0 + rows_per_chunk), device=dev)
        w = weights(slices, rows, c)  # [n, m]
        if not (w > 0).any():
            continue
        qs, dos = q[rows].float(), do[rows].float()
        s = torch.einsum("nhd,mhd->hnm", qs, kf) * scale
        lse = lse_all[:, rows]
        p = torch.exp(s - torch.where(torch.isfinite(lse), lse, 0)[..., None]) * w[None]
        dp = torch.einsum("nhd,mhd->hnm", dos, vf)
        ds = p * (dp - delta_all[rows].T[..., None])
        dv += torch.einsum("hnm,nhd->mhd", p, dos)
        dk += torch.einsum("hnm,nhd->mhd", ds, qs) * scale
    return dk.reshape(len(keys), hk, grp, d).sum(2), dv.reshape(len(keys), hk, grp, d).sum(2)


def max_err(got: torch.Tensor, ref: torch.Tensor) -> tuple[float, float]:
    """(max abs error, max abs error / max |ref|) over finite reference entries."""
    got, ref = got.double(), ref.double()
    fin = torch.isfinite(ref)
    if not fin.any():
        return 0.0, 0.0
    diff = (got[fin] - ref[fin]).abs().max().item()
    return diff, diff / max(ref[fin].abs().max().item(), 1e-12)
