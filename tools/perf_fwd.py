"""Quick FFA kernel timing (development helper; bench.py is the contract)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_13211_b200.ffa import FFAPlan, ffa_backward, ffa_forward  # noqa: E402


def block_causal(s, b):
    return [[i, i + b] for i in range(0, s, b)], [[0, i + b] for i in range(0, s, b)], [0] * (s // b)


def run(s, hq, hk, d, block, bwd=False, iters=10):
    qr, kr, ty = block_causal(s, block)
    plan = FFAPlan(qr, kr, ty, s, s, d)
    area = plan.area()
    q = torch.randn(s, hq, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(s, hk, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(s, hk, d, device="cuda", dtype=torch.bfloat16)
    do = torch.randn(s, hq, d, device="cuda", dtype=torch.bfloat16)
    out, lse = ffa_forward(plan, q, k, v)
    for _ in range(3):
        ffa_forward(plan, q, k, v, out=out, lse=lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ffa_forward(plan, q, k, v, out=out, lse=lse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 4 * area * hq * d
    print(f"fwd S={s} hq={hq} hk={hk} d={d} block={block}: {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOPS")
    if bwd:
        try:
            for _ in range(2):
                ffa_backward(plan, q, k, v, out, lse, do)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(iters):
                ffa_backward(plan, q, k, v, out, lse, do)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / iters
            print(f"bwd: {ms:.3f} ms, {2.5 * fl / ms / 1e9:.1f} TFLOPS")
        except Exception as e:  # noqa: BLE001
            print("bwd failed:", e)


if __name__ == "__main__":
    run(1024, 1, 1, 64, 256)
    run(32768, 24, 8, 128, 4096, bwd=True)
    run(32768, 48, 8, 128, 4096, bwd=True)
    run(32768, 48, 8, 128, 2048)
