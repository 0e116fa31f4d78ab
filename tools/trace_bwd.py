"""Timeline of one dK/dV CTA (diagnostics; see magiplan_debug_set_trace).

Per-role logs (globaltimer ns): MMA 1 = P^T(t) ready, 2 = Q(t+1) landed,
3 = dS^T(t) ready, 4 = dO(t+1) landed; warpgroups 10..13 = S(t) ready, P^T
written, dP(t) ready, dS^T(t) written; TMA 30 / 31 = Q / dO slot for step t free.
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_13211_b200 import _lib  # noqa: E402

# the diagnostics build (python -m paper_2505_13211_b200.build --trace), or MAGI_LIB
_lib._LIB_PATH = _lib.Path(os.environ.get("MAGI_LIB", "build/trace/libmagiplan.so")).resolve()
from paper_2505_13211_b200.ffa import FFAPlan, ffa_backward, ffa_forward  # noqa: E402

CAP = 8000


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
    buf = torch.zeros(1 + 5 * 2 * CAP, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().magiplan_debug_set_trace(buf.data_ptr(), block))
    ffa_backward(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().magiplan_debug_set_trace(None, 0))
    data = buf[1:].view(5, CAP, 2)[:4].cpu().tolist()
    ev = {}
    for role in range(4):
        for key, ns in data[role]:
            if ns == 0:
                break
            ev.setdefault((key >> 32, key & 0xFFFFFFFF), ns)
    if any(k[0] == 98 for k in ev) and any(k[0] == 99 for k in ev):
        (c0k, n0), = [(k, v) for k, v in ev.items() if k[0] == 98]
        (c1k, n1), = [(k, v) for k, v in ev.items() if k[0] == 99]
        dc = (c1k[1] - c0k[1]) % (1 << 32)
        print(f"SM clock during the traced CTA: {dc / max(n1 - n0, 1) * 1e3:.0f} MHz")
    ev = {k: v for k, v in ev.items() if k[0] < 90}
    steps = max(t for _, t in ev) + 1
    t0 = min(ev.values())

    def gap(a, b, off=0):
        xs = [ev[(b, t)] - ev[(a, t + off)] for t in range(2, steps - 2) if (a, t + off) in ev and (b, t) in ev]
        return statistics.median(xs) if xs else float("nan")

    per = [ev[(3, t + 1)] - ev[(3, t)] for t in range(2, steps - 3) if (3, t + 1) in ev and (3, t) in ev]
    print(f"block {block}: {steps} steps, span {(max(ev.values()) - t0) / 1e3:.1f} us, "
          f"step period median {statistics.median(per):.0f} ns")
    for w in (0, 1):
        print(f"wg{w}: S ready->P written {gap(10, 11):.0f} | P->dP ready {gap(11, 12):.0f} | "
              f"dP ready->dS written {gap(12, 13):.0f} | dS written(t-1)->S ready(t) {gap(13, 10, -1):.0f} ns")
    print(f"exp phase: S ready->S in regs {gap(10, 14):.0f} | ->P packed {gap(14, 15):.0f} | "
          f"->P stored {gap(15, 16):.0f} | ->arrived {gap(16, 11):.0f} ns")
    print(f"mma: P ready->Q(t+1) landed {gap(1, 2):.0f} | Q landed->dS ready {gap(2, 3):.0f} | "
          f"dS ready->dO(t+1) landed {gap(3, 4):.0f} ns")
    for t in range(3, min(steps, 6)):
        row = [f"{e}:{(ev[(e, t)] - t0) / 1e3:.2f}" for e in (30, 31, 1, 2, 3, 4, 10, 11, 12, 13) if (e, t) in ev]
        print(f"  t={t} " + " ".join(row))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
