"""Host tile planner -> kernel contract (CPU).

For every slice list the q-major work lists (128- and 256-row tiles) must
cover each allowed (q, k) pair of their rows exactly as often as the mask's
multiplicity says, once the kernel's per-row bounds are applied inside the
listed key tiles; likewise the k-major list for the dK/dV kernel. Rows that
no slice touches still get a tile (they are written as empty rows)."""
import numpy as np
import pytest

from tests.ffa_cases import CASES


def _bounds(qs, qe, ks, ke, ty, q):
    if q < qs or q >= qe:
        return 0, 0
    lo = min(ks + (q - qs), ke) if ty in (2, 3) else ks
    hi = min(max(q + ke - qe + 1, ks), ke) if ty in (1, 3) else ke
    return lo, hi


def _slices(case):
    sq, sk, hq, hk, d, qr, kr, ty = CASES[case]
    return sq, sk, d, [[*q, *k, t] for q, k, t in zip(qr, kr, ty)]


@pytest.mark.parametrize("case", sorted(CASES))
def test_worklists_cover_mask_exactly(built_lib, case):
    from oracle import oracle
    from paper_2505_13211_b200.planner import debug_eval

    sq, sk, d, sl = _slices(case)
    wl = debug_eval("ffa_worklists", seqlen_q=sq, seqlen_k=sk, head_dim=d, slices=sl)
    want = oracle.dense_allowed(sq, sk, [s[0:2] for s in sl], [s[2:4] for s in sl], [s[4] for s in sl])
    assert wl["area_multiplicity"] == int(want.sum())
    for key, rows in (("fwd128", 128), ("fwd256", 256)):
        got = np.zeros_like(want)
        seen_rows = set()
        for tile in wl[key]:
            q0 = tile["q0"]
            seen_rows.add(q0)
            assert tile["n_ktiles"] == sum(it[6] for it in tile["items"])
            for qs, qe, ks, ke, ty, kb, nk in tile["items"]:
                for q in range(q0, min(q0 + rows, sq)):
                    lo, hi = _bounds(qs, qe, ks, ke, ty, q)
                    for k in range(kb, kb + nk * 128):
                        if lo <= k < hi:
                            got[q, k] += 1
        np.testing.assert_array_equal(got, want)
        assert seen_rows == set(range(0, sq, rows))
        w = [t["n_ktiles"] for t in wl[key]]
        assert w == sorted(w, reverse=True)  # LPT order
    got = np.zeros_like(want)
    for tile in wl["bwd"]:
        k0 = tile["k0"]
        for qs, qe, ks, ke, ty, qb, nq in tile["items"]:
            for q in range(qb, min(qb + nq * 128, sq)):
                lo, hi = _bounds(qs, qe, ks, ke, ty, q)
                for k in range(k0, min(k0 + 128, sk)):
                    if lo <= k < hi:
                        got[q, k] += 1
    np.testing.assert_array_equal(got, want)
