"""Timeline of one dQ CTA (diagnostics: a library built with
`python -m paper_2505_13211_b200.build --trace`; magiplan_debug_set_trace with
a negative block index -b-1 selects dQ CTA b).

MMA 1 = S slot free (S(t) in registers), 2 = dS(t) ready (p_full), 3 = dP(t+1)
issued; warpgroups 10 = S(t) ready, 11 = exponentials done, 12 = dP(t) ready,
13 = dS(t) written.
"""
import os
import statistics
import sys

import torch  # noqa: E402

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
    _lib.check(_lib.lib().magiplan_debug_set_trace(buf.data_ptr(), -block - 1))
    ffa_backward(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().magiplan_debug_set_trace(None, 0))
    data = buf[1:].view(5, CAP, 2)[:3].cpu().tolist()
    ev = {}
    for role in range(3):
        for key, ns in data[role]:
            if ns == 0:
                break
            ev.setdefault((key >> 32, key & 0xFFFFFFFF), ns)
    if any(k[0] == 98 for k in ev) and any(k[0] == 99 for k in ev):
        (c0k, n0), = [(k, v) for k, v in ev.items() if k[0] == 98]
        (c1k, n1), = [(k, v) for k, v in ev.items() if k[0] == 99]
        print(f"SM clock: {((c1k[1] - c0k[1]) % (1 << 32)) / max(n1 - n0, 1) * 1e3:.0f} MHz")
    ev = {k: v for k, v in ev.items() if k[0] < 90}
    steps = max(t for _, t in ev) + 1
    t0 = min(ev.values())

    def gap(a, b, off=0):
        xs = [ev[(b, t)] - ev[(a, t + off)] for t in range(2, steps - 2) if (a, t + off) in ev and (b, t) in ev]
        return statistics.median(xs) if xs else float("nan")

    per = [ev[(2, t + 1)] - ev[(2, t)] for t in range(2, steps - 3) if (2, t + 1) in ev and (2, t) in ev]
    print(f"block {block}: {steps} steps, step period median {statistics.median(per):.0f} ns")
    print(f"wg: S ready->exp done {gap(10, 11):.0f} | exp done->dP ready {gap(11, 12):.0f} | "
          f"dP ready->dS written {gap(12, 13):.0f} | dS written(t-1)->S ready(t) {gap(13, 10, -1):.0f} ns")
    print(f"mma: dS ready(t)->dP(t+1) issued {gap(2, 3):.0f} | dP issued(t)->S free(t+1) {gap(3, 1, -1):.0f} | "
          f"S free->dS ready {gap(1, 2):.0f} ns")
    for t in range(3, min(steps, 7)):
        row = [f"{e}:{(ev[(e, t)] - t0) / 1e3:.2f}" for e in (1, 2, 3, 10, 11, 12, 13) if (e, t) in ev]
        print(f"  t={t} " + " ".join(row))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
