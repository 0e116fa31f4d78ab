"""A/B (development helper): the two backward passes serialised on one stream
vs dQ forked onto a second stream so its CTAs fill the SMs the dK/dV pass
drains (the passes are independent: both read Q, K, V, dO, LSE, delta).

    python tools/overlap_bwd.py          # config 2 (S 32768, block 4096, 24q/8kv)
"""
import math
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_13211_b200 import _lib  # noqa: E402
from paper_2505_13211_b200.ffa import FFAPlan  # noqa: E402


def main(S=32768, hq=24, hk=8, d=128, block=4096, iters=10):
    dev = torch.device("cuda", 0)
    qr = [[b, b + block] for b in range(0, S, block)]
    kr = [[0, b + block] for b in range(0, S, block)]
    plan = FFAPlan(qr, kr, [0] * len(qr), S, S, d)
    q = torch.randn(S, hq, d, device=dev, dtype=torch.bfloat16)
    k = torch.randn(S, hk, d, device=dev, dtype=torch.bfloat16)
    v = torch.randn(S, hk, d, device=dev, dtype=torch.bfloat16)
    do = torch.randn(S, hq, d, device=dev, dtype=torch.bfloat16)
    out = torch.empty_like(q)
    lse = torch.empty(hq, S, device=dev)
    delta = torch.empty(hq, S, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    L, BF, scale = _lib.lib(), _lib.BF16, 1.0 / math.sqrt(d)
    s0 = torch.cuda.current_stream(dev)
    s1 = torch.cuda.Stream(dev)

    def fwd_pre(sp):
        _lib.check(L.magiplan_ffa_fwd(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                      lse.data_ptr(), hq, hk, scale, BF, 0, sp))
        _lib.check(L.magiplan_ffa_bwd_preprocess(out.data_ptr(), do.data_ptr(), delta.data_ptr(), S, hq, d, BF, sp))

    def dkdv(sp):
        _lib.check(L.magiplan_ffa_bwd_dkdv(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), lse.data_ptr(),
                                           delta.data_ptr(), do.data_ptr(), dk.data_ptr(), dv.data_ptr(), hq, hk,
                                           scale, BF, 0, sp))

    def dqp(sp):
        _lib.check(L.magiplan_ffa_bwd_dq(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), lse.data_ptr(),
                                         delta.data_ptr(), do.data_ptr(), dq.data_ptr(), hq, hk, scale, BF, 0, sp))

    def step(mode):
        fwd_pre(s0.cuda_stream)
        if mode == "serial":
            dkdv(s0.cuda_stream)
            dqp(s0.cuda_stream)
        else:
            e = torch.cuda.Event()
            e.record(s0)
            s1.wait_event(e)
            first, second = (dkdv, dqp) if mode == "fork_dq" else (dqp, dkdv)
            first(s0.cuda_stream)
            second(s1.cuda_stream)
            j = torch.cuda.Event()
            j.record(s1)
            s0.wait_event(j)

    res = {}
    for mode in ["serial", "fork_dq", "fork_dkdv"] * 2:
        for _ in range(3):
            step(mode)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s0)
        for _ in range(iters):
            step(mode)
        b.record(s0)
        torch.cuda.synchronize()
        res.setdefault(mode, []).append(a.elapsed_time(b) / iters)
    for mode, xs in res.items():
        print(f"{mode:10s} step ms {[round(x, 3) for x in xs]}  median {statistics.median(xs):.3f}")
    # the forked results must equal the serial ones bit for bit
    step("serial")
    torch.cuda.synchronize()
    ref = [t.clone() for t in (dq, dk, dv)]
    step("fork_dq")
    torch.cuda.synchronize()
    print("fork bitwise equal:", all(torch.equal(x, y) for x, y in zip(ref, (dq, dk, dv))))


if __name__ == "__main__":
    main()
