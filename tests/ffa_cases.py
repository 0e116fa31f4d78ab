"""Slice-list cases shared by the FFA parity tests (GPU vs the CPU oracle)."""
from __future__ import annotations

import numpy as np
import torch

FULL, CAUSAL, INV, BI = 0, 1, 2, 3


def block_causal(seqlen, block):
    qr = [[b, b + block] for b in range(0, seqlen, block)]
    kr = [[0, b + block] for b in range(0, seqlen, block)]
    return qr, kr, [FULL] * len(qr)


def varlen(lengths, types):
    qr, kr, off = [], [], 0
    for n in lengths:
        qr.append([off, off + n])
        kr.append([off, off + n])
        off += n
    return qr, kr, list(types)


def random_slices(sq, sk, n, seed):
    """n random (possibly overlapping, possibly non-square) slices of all four
    types: MULTIPLICITY semantics and the diagonal anchors of every type on
    tiles that start and end mid-tile."""
    rng = np.random.default_rng(seed)
    qr, kr, ty = [], [], []
    while len(qr) < n:
        a, b = sorted(int(x) for x in rng.integers(0, sq + 1, 2))
        c, e = sorted(int(x) for x in rng.integers(0, sk + 1, 2))
        if b - a < 1 or e - c < 1:
            continue
        qr.append([a, b])
        kr.append([c, e])
        ty.append(int(rng.integers(0, 4)))
    return qr, kr, ty


# name -> (sq, sk, hq, hk, d, q_ranges, k_ranges, types)
CASES = {
    "cfg1_block_causal_d64": (1024, 1024, 1, 1, 64, *block_causal(1024, 256)),
    "block_causal_gqa_d128": (1024, 1024, 4, 2, 128, *block_causal(1024, 256)),
    "causal_unaligned": (300, 300, 2, 1, 128, [[0, 300]], [[0, 300]], [CAUSAL]),
    "varlen_mixed": (512, 512, 2, 2, 128, *varlen([100, 37, 250, 125], [FULL, CAUSAL, FULL, CAUSAL])),
    "inv_bi_d64": (384, 384, 2, 1, 64, [[0, 200], [200, 384]], [[0, 384], [50, 300]], [INV, BI]),
    "overlap_multiplicity": (256, 256, 2, 2, 128, [[0, 256], [64, 192]], [[0, 256], [32, 160]],
                             [FULL, CAUSAL]),
    "empty_rows": (256, 256, 1, 1, 128, [[0, 100]], [[0, 256]], [FULL]),
    "cross_lk_gt_lq": (200, 520, 2, 2, 128, [[0, 120], [120, 200]], [[0, 520], [100, 400]],
                       [FULL, CAUSAL]),
    "causal_lq_gt_lk": (400, 300, 1, 1, 64, [[0, 400]], [[0, 300]], [CAUSAL]),
    "sliding_window": (640, 640, 2, 1, 128, [[0, 96], [96, 640]], [[0, 96], [1, 640]], [CAUSAL, BI]),
    # keys [0,128), [300,400), [450,512) in no slice: dK/dV must come back 0
    # a PnP-packed bin (planner.packed_bin_masks(lognormal_lengths(200, 150, 0.8,
    # 1024, 5), 1024, 2, pool_capacity=32)[3]): 5 documents, 7-row padding tail
    "packed_bin_padding_tail": (1024, 1024, 4, 2, 128,
                                *varlen([299, 237, 222, 200, 59], [FULL, CAUSAL, FULL, CAUSAL, FULL])),
    "uncovered_keys": (256, 512, 2, 1, 128, [[0, 256], [0, 100]], [[128, 300], [400, 450]],
                       [FULL, CAUSAL]),
    # zero-length q or k ranges next to real slices (legal: qs <= qe, ks <= ke)
    "degenerate_slices": (300, 300, 2, 2, 128, [[50, 50], [0, 300], [10, 200]],
                          [[0, 300], [0, 300], [77, 77]], [FULL, CAUSAL, BI]),
    # an empty slice list: every row empty, every gradient 0
    "no_slices": (192, 192, 1, 1, 128, [], [], []),
    # 41 short documents (1..31 tokens) in one packed sequence, GQA 4:1
    "many_tiny_docs": (641, 641, 4, 1, 128,
                       *varlen([1 + (7 * i) % 31 for i in range(41)], [i % 2 for i in range(41)])),
    # GQA 6:1 at head_dim 64, unaligned causal
    "gqa6_causal_d64": (333, 333, 6, 1, 64, [[0, 333]], [[0, 333]], [CAUSAL]),
    # GQA 16:1 (a single kv head): the dK/dV pass walks 16 q heads per key tile
    "gqa16_block_causal": (512, 512, 16, 1, 128, *block_causal(512, 128)),
    # 12 random overlapping slices of all four types, sq != sk
    "random_overlapping": (700, 900, 2, 1, 128, *random_slices(700, 900, 12, seed=2025)),
}


def make_inputs(sq, sk, hq, hk, d, seed=0, device="cuda"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    q = torch.randn(sq, hq, d, generator=g).to(torch.bfloat16)
    k = torch.randn(sk, hk, d, generator=g).to(torch.bfloat16)
    v = torch.randn(sk, hk, d, generator=g).to(torch.bfloat16)
    do = torch.randn(sq, hq, d, generator=g).to(torch.bfloat16)
    return q.to(device), k.to(device), v.to(device), do.to(device)


def err_stats(got: np.ndarray, ref: np.ndarray) -> tuple[float, float]:
    """(max abs error, max abs error / max |ref|) over finite reference entries."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    fin = np.isfinite(ref)
    if not fin.any():
        return 0.0, 0.0
    diff = np.abs(got[fin] - ref[fin])
    scale = max(np.abs(ref[fin]).max(), 1e-12)
    return float(diff.max()), float(diff.max() / scale)
