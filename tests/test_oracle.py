"""Pins the CPU FFA oracle (oracle/ffa_oracle.c) before it is trusted:
  1. its slice membership reproduces the reference planner's row unions and
     MULTIPLICITY areas on every golden mask (tests/golden, generated from
     the compiled reference);
  2. its numerics match an independent dense float64 torch formulation
     (softmax over a multiplicity-weighted mask; autograd for gradients).
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle

GOLD = json.loads((Path(__file__).parent / "golden" / "ref_planner.json").read_text())


def _slices(mask_json):
    qr = [s["q"] for s in mask_json["slices"]]
    kr = [s["k"] for s in mask_json["slices"]]
    ty = [{"full": 0, "causal": 1, "inv_causal": 2, "bi_causal": 3}[s["type"]] for s in mask_json["slices"]]
    return qr, kr, ty


def test_oracle_membership_matches_reference_masks():
    cases = [(e["json"], e["row_counts"], e["area_multiplicity"]) for e in GOLD["named_masks"]
             if "row_counts" in e and e["json"]["seqlen_q"] <= 128]
    cases += [(e["mask"], e["row_counts"], e["area_multiplicity"]) for e in GOLD["random_masks"]]
    assert len(cases) > 50
    for mj, rows, mult in cases:
        qr, kr, ty = _slices(mj)
        cnt = oracle.dense_allowed(mj["seqlen_q"], mj["seqlen_k"], qr, kr, ty)
        assert int(cnt.sum()) == mult
        assert [int(x) for x in (cnt > 0).sum(axis=1)] == rows


def _dense_reference(q, k, v, do, qr, kr, ty, scale):
    sq, hq, d = q.shape
    sk, hk, _ = k.shape
    cnt = oracle.dense_allowed(sq, sk, qr, kr, ty).astype(np.float64)
    W = torch.from_numpy(cnt)  # multiplicity weights
    qd = q.double().requires_grad_(True)
    kd = k.double().requires_grad_(True)
    vd = v.double().requires_grad_(True)
    g = hq // hk
    kr_ = kd.repeat_interleave(g, dim=1)
    vr_ = vd.repeat_interleave(g, dim=1)
    s = torch.einsum("qhd,khd->hqk", qd, kr_) * scale
    m = torch.where(W > 0, s, torch.tensor(-math.inf, dtype=torch.float64)).amax(-1, keepdim=True)
    m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
    e = torch.exp(s - m) * W
    l = e.sum(-1, keepdim=True)
    l_safe = torch.where(l > 0, l, torch.ones_like(l))  # empty rows: e == 0 -> p == 0, no NaN grads
    p = e / l_safe
    o = torch.einsum("hqk,khd->qhd", p, vr_)
    lse = torch.where(l[..., 0] > 0, m[..., 0] + torch.log(l_safe[..., 0]),
                      torch.tensor(-math.inf, dtype=torch.float64))
    o.backward(do.double())
    return o.detach().numpy(), lse.detach().numpy(), qd.grad.numpy(), kd.grad.numpy(), vd.grad.numpy()


@pytest.mark.parametrize("case", ["overlap", "gqa_causal", "inv_bi", "empty_rows"])
def test_oracle_numerics_vs_dense_float64(case):
    torch.manual_seed(0)
    d = 16
    if case == "overlap":
        sq = sk = 48
        hq = hk = 2
        qr, kr, ty = [[0, 48], [8, 40]], [[0, 48], [4, 30]], [0, 1]
    elif case == "gqa_causal":
        sq, sk, hq, hk = 40, 56, 4, 2
        qr, kr, ty = [[0, 40]], [[0, 56]], [1]
    elif case == "inv_bi":
        sq = sk = 50
        hq, hk = 2, 1
        qr, kr, ty = [[0, 25], [25, 50]], [[0, 50], [10, 40]], [2, 3]
    else:
        sq = sk = 32
        hq = hk = 1
        qr, kr, ty = [[0, 10]], [[0, 32]], [0]
    q = torch.randn(sq, hq, d).to(torch.bfloat16).float()
    k = torch.randn(sk, hk, d).to(torch.bfloat16).float()
    v = torch.randn(sk, hk, d).to(torch.bfloat16).float()
    do = torch.randn(sq, hq, d).to(torch.bfloat16).float()
    scale = 1 / math.sqrt(d)
    o, lse = oracle.ffa_fwd(q, k, v, qr, kr, ty, scale)
    dq, dk, dv = oracle.ffa_bwd(q, k, v, o, lse, do, qr, kr, ty, scale)
    ro, rl, rdq, rdk, rdv = _dense_reference(q, k, v, do, qr, kr, ty, scale)
    np.testing.assert_allclose(o, ro, atol=1e-10)
    fin = np.isfinite(rl)
    np.testing.assert_allclose(lse[fin], rl[fin], atol=1e-10)
    assert np.all(np.isneginf(lse[~fin]))
    np.testing.assert_allclose(dq, rdq, atol=1e-9)
    np.testing.assert_allclose(dk, rdk, atol=1e-9)
    np.testing.assert_allclose(dv, rdv, atol=1e-9)
    # the f32-accumulating variant used for the CPU baseline agrees to f32 precision
    of, lf = oracle.ffa_fwd(q, k, v, qr, kr, ty, scale, acc_f32=True)
    np.testing.assert_allclose(of, o, atol=1e-5)


@pytest.mark.parametrize("name", ["varlen_mixed", "inv_bi_d64", "overlap_multiplicity", "empty_rows",
                                  "cross_lk_gt_lq", "causal_lq_gt_lk", "uncovered_keys", "sliding_window"])
def test_dense_fp32_reference_matches_oracle(name):
    """tests/dense_ref.py (the full-size GPU tests' fp32 reference, which
    recomputes LSE / O / delta itself) agrees with the pinned oracle on the
    slice-list edge cases: multiplicity, INV/BI types, empty rows, keys no
    slice reaches, cross-length slices. Run on CPU here."""
    from tests import dense_ref
    from tests.ffa_cases import CASES, make_inputs

    sq, sk, hq, hk, d, qr, kr, ty = CASES[name]
    q, k, v, do = make_inputs(sq, sk, hq, hk, d, seed=3, device="cpu")
    scale = 1.0 / math.sqrt(d)
    ro, rl = oracle.ffa_fwd(q, k, v, qr, kr, ty, scale)
    rdq, rdk, rdv = oracle.ffa_bwd(q, k, v, ro, rl, do, qr, kr, ty, scale)
    slices = [(tuple(a), tuple(b), t) for a, b, t in zip(qr, kr, ty)]
    out, lse = dense_ref.forward_all(q, k, v, slices, scale, rows_per_chunk=64)
    rows, keys = list(range(0, sq, 7)), list(range(0, sk, 5))
    o, l, dq = dense_ref.rows_ref(q, k, v, do, slices, scale, rows, lse, out)
    dk, dv = dense_ref.keys_ref(q, k, v, do, slices, scale, keys, lse, out, rows_per_chunk=64)
    fin = np.isfinite(rl)
    assert np.array_equal(np.isfinite(lse.numpy()), fin)
    assert np.abs(lse.numpy()[fin] - rl[fin]).max() < 1e-5
    for got, ref in ((out.numpy(), ro), (dq.numpy(), rdq[rows]), (dk.numpy(), rdk[keys]),
                     (dv.numpy(), rdv[keys])):
        assert np.abs(got - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("name", ["cfg1_block_causal_d64", "block_causal_gqa_d128", "causal_unaligned",
                                  "varlen_mixed", "inv_bi_d64", "empty_rows", "cross_lk_gt_lq",
                                  "causal_lq_gt_lk", "sliding_window", "uncovered_keys", "many_tiny_docs",
                                  "gqa6_causal_d64", "gqa16_block_causal"])
def test_oracle_matches_torch_sdpa(name):
    """A third, external pin of the oracle's numerics: PyTorch's own
    scaled_dot_product_attention (float64, math kernel, autograd) with the
    boolean mask of the slice list (membership from the reference-pinned
    oracle.dense_allowed), on every case whose slices do not overlap (SDPA
    has no multiplicity). Rows without keys are left out (SDPA returns NaN
    there; their dO is zeroed so they add nothing to dK / dV)."""
    import torch.nn.functional as F

    from tests.ffa_cases import CASES, make_inputs

    sq, sk, hq, hk, d, qr, kr, ty = CASES[name]
    cnt = oracle.dense_allowed(sq, sk, qr, kr, ty)
    assert cnt.max() <= 1, "overlapping slices: not expressible as an SDPA mask"
    q, k, v, do = make_inputs(sq, sk, hq, hk, d, seed=4, device="cpu")
    scale = 1.0 / math.sqrt(d)
    ro, rl = oracle.ffa_fwd(q, k, v, qr, kr, ty, scale)
    rdq, rdk, rdv = oracle.ffa_bwd(q, k, v, ro, rl, do, qr, kr, ty, scale)

    has = cnt.sum(axis=1) > 0
    mask = torch.from_numpy(cnt > 0)
    mask[~torch.from_numpy(has)] = True  # keep SDPA finite on empty rows (excluded below)
    g = hq // hk
    qd = q.double().permute(1, 0, 2).requires_grad_(True)            # [hq, sq, d]
    kd = k.double().permute(1, 0, 2).requires_grad_(True)            # [hk, sk, d]
    vd = v.double().permute(1, 0, 2).requires_grad_(True)
    o = F.scaled_dot_product_attention(qd, kd.repeat_interleave(g, 0), vd.repeat_interleave(g, 0),
                                       attn_mask=mask, scale=scale)
    dod = do.double().permute(1, 0, 2) * torch.from_numpy(has)[None, :, None]
    o.backward(dod)
    o = o.detach().permute(1, 0, 2).numpy()
    sdq = qd.grad.permute(1, 0, 2).numpy()
    sdk = kd.grad.permute(1, 0, 2).numpy()
    sdv = vd.grad.permute(1, 0, 2).numpy()
    tol = 1e-9 * max(1.0, float(np.abs(ro).max()))
    assert np.abs(o[has] - ro[has]).max() <= tol
    assert np.all(ro[~has] == 0) and np.all(np.isneginf(rl[:, ~has]))
    assert np.abs(sdq[has] - rdq[has]).max() <= 1e-9 * max(1.0, float(np.abs(rdq).max()))
    assert np.abs(sdk - rdk).max() <= 1e-9 * max(1.0, float(np.abs(rdk).max()))
    assert np.abs(sdv - rdv).max() <= 1e-9 * max(1.0, float(np.abs(rdv).max()))

