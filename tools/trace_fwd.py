"""Timeline of one forward CTA (diagnostics; see magiplan_debug_set_trace).

Per-role logs (globaltimer ns): MMA 1 = P0(t) ready, 2 = V(t) landed,
3 = K(t+1) landed, 4 = P1(t) ready; softmax warpgroups 10..13 = S(t) ready,
S in registers, exp done, P(t) written; TMA 30 / 31 = K / V slot for tile t free.
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_13211_b200 import _lib  # noqa: E402

# the diagnostics build (python -m paper_2505_13211_b200.build --trace), or MAGI_LIB
_lib._LIB_PATH = _lib.Path(os.environ.get("MAGI_LIB", "build/trace/libmagiplan.so")).resolve()
from paper_2505_13211_b200.ffa import FFAPlan, ffa_forward  # noqa: E402

CAP = 8000


def main(block: int = 0):
    S, hq, hk, d, b = 32768, 24, 8, 128, 4096
    qr = [[i, i + b] for i in range(0, S, b)]
    kr = [[0, i + b] for i in range(0, S, b)]
    plan = FFAPlan(qr, kr, [0] * len(qr), S, S, d)
    q = torch.randn(S, hq, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(S, hk, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(S, hk, d, device="cuda", dtype=torch.bfloat16)
    ffa_forward(plan, q, k, v)
    buf = torch.zeros(1 + 5 * 2 * CAP, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().magiplan_debug_set_trace(buf.data_ptr(), block))
    ffa_forward(plan, q, k, v)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().magiplan_debug_set_trace(None, 0))
    data = buf[1:].view(5, CAP, 2).cpu().tolist()
    ev = {}
    for role in range(5):
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

    per = [ev[(1, t + 1)] - ev[(1, t)] for t in range(2, steps - 3) if (1, t + 1) in ev and (1, t) in ev]
    print(f"block {block}: {steps} key tiles, span {(max(ev.values()) - t0) / 1e3:.1f} us, "
          f"period median {statistics.median(per):.0f} ns (MMA-only bound ~1050 ns at 1.96 GHz)")
    print("softmax WG0 events are 10..13 of role 1, WG1 of role 2 (both keyed the same; role 1 wins)")
    print(f"S ready->in regs {gap(10, 11):.0f} | regs->exp done {gap(11, 12):.0f} | "
          f"exp->P written {gap(12, 13):.0f} | P written(t-1)->S ready(t) {gap(13, 10, -1):.0f} ns")
    print(f"K load latency (slot free -> landed) {gap(30, 32):.0f} | V {gap(31, 33):.0f} ns")
    print(f"mma: P0 ready->V landed {gap(1, 2):.0f} | V->K(t+1) landed {gap(2, 3):.0f} | "
          f"K(t+1)->P1 ready {gap(3, 4):.0f} | P1(t)->P0(t+1) {gap(4, 1, -1):.0f} ns")
    for t in range(3, min(steps, 7)):
        row = [f"{e}:{(ev[(e, t)] - t0) / 1e3:.2f}" for e in (30, 31, 32, 33, 1, 2, 3, 4, 10, 11, 12, 13) if (e, t) in ev]
        print(f"  t={t} " + " ".join(row))
    # both warpgroups separately
    for role in (1, 2):
        evr = {}
        for key, ns in data[role]:
            if ns == 0:
                break
            evr[(key >> 32, key & 0xFFFFFFFF)] = ns

        def g2(a, b, off=0):
            xs = [evr[(b, t)] - evr[(a, t + off)] for t in range(2, steps - 2)
                  if (a, t + off) in evr and (b, t) in evr]
            return statistics.median(xs) if xs else float("nan")

        print(f"WG{role - 1}: S ready->ld done {g2(10, 14):.0f} | ->max stored {g2(14, 15):.0f} | "
              f"->barrier passed {g2(15, 11):.0f} | ->exp done {g2(11, 12):.0f} | "
              f"exp->P written {g2(12, 13):.0f} | P written(t-1)->S ready(t) {g2(13, 10, -1):.0f} ns")
        print("   " + " ".join(f"{(evr[(10, t)] - t0) / 1e3:.2f}/{(evr[(13, t)] - t0) / 1e3:.2f}"
                           for t in range(3, min(steps, 9)) if (10, t) in evr and (13, t) in evr))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
