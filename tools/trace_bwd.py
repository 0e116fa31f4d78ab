"""Timeline of one dK/dV CTA (diagnostics; see magiplan_debug_set_trace).

Events (globaltimer ns): MMA warp 1 = S(t+1) slot free, 2 = Q/dO(t+1) landed,
3 = P/dS(t) ready; warpgroup w (10*w+10..13): S(t) ready, exp done, dP(t)
ready, P/dS(t) written.
"""
import math
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_13211_b200 import _lib  # noqa: E402
from paper_2505_13211_b200.ffa import FFAPlan, ffa_backward, ffa_forward  # noqa: E402


def main(block: int = 0):
    S, hq, hk, d, b = 32768, 24, 8, 128, 4096
    qr = [[i, i + b] for i in range(0, S, b)]
    kr = [[0, i + b] for i in range(0, S, b)]
    plan = FFAPlan(qr, kr, [0] * len(qr), S, S, d)
    q = torch.randn(S, hq, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(S, hk, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(S, hk, d, device="cuda", dtype=torch.bfloat16)
    do = torch.randn(S, hq, d, device="cuda", dtype=torch.bfloat16)
    out, lse = ffa_forward(plan, q, k, v)
    ffa_backward(plan, q, k, v, out, lse, do)
    buf = torch.zeros(1 + 3 * 20000, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().magiplan_debug_set_trace(buf.data_ptr(), block))
    ffa_backward(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().magiplan_debug_set_trace(None, 0))
    n = int(buf[0])
    rec = buf[1:1 + 3 * min(n, 20000)].view(-1, 3).cpu().tolist()
    ev = {}
    for e, t, ns in rec:
        ev.setdefault((e, t), ns)
    steps = max(t for _, t in ev) + 1
    t0 = min(ns for ns in ev.values())

    def gap(a, b, ta_off=0):
        out = []
        for t in range(1, steps - 1):
            if (a, t + ta_off) in ev and (b, t) in ev:
                out.append(ev[(b, t)] - ev[(a, t + ta_off)])
        return statistics.median(out) if out else float("nan")

    print(f"block {block}: {n} records, {steps} steps, span {(max(ev.values()) - t0) / 1e3:.1f} us")
    per = [ev[(3, t + 1)] - ev[(3, t)] for t in range(1, steps - 2) if (3, t + 1) in ev and (3, t) in ev]
    print(f"step period (P ready -> next P ready): median {statistics.median(per):.0f} ns")
    for w in (0, 1):
        base = 10 + 10 * w
        print(f"wg{w}: S ready->exp done {gap(base, base + 1):.0f} ns | exp done->dP ready "
              f"{gap(base + 1, base + 2):.0f} | dP ready->P/dS written {gap(base + 2, base + 3):.0f} | "
              f"P/dS written(t-1)->S ready(t) {gap(base + 3, base, -1):.0f}")
    print(f"mma: S-slot free->Q/dO landed {gap(1, 2):.0f} ns | Q/dO landed(t)->P ready(t) {gap(2, 3):.0f} ns")
    for t in range(2, min(steps, 6)):
        row = [f"{e}:{(ev[(e, t)] - t0) / 1e3:.2f}" for e in (1, 2, 3, 10, 11, 12, 13, 20, 21, 22, 23) if (e, t) in ev]
        print(f"  t={t} " + " ".join(row))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
