"""One forward + backward pass at config 2 shapes (for ncu captures: exactly
one launch of each FFA kernel)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_13211_b200.ffa import FFAPlan, ffa_backward, ffa_forward  # noqa: E402

S, HQ, HK, D, B = 32768, 24, 8, 128, 4096
qr = [[i, i + B] for i in range(0, S, B)]
kr = [[0, i + B] for i in range(0, S, B)]
plan = FFAPlan(qr, kr, [0] * len(qr), S, S, D)
q = torch.randn(S, HQ, D, device="cuda", dtype=torch.bfloat16)
k = torch.randn(S, HK, D, device="cuda", dtype=torch.bfloat16)
v = torch.randn(S, HK, D, device="cuda", dtype=torch.bfloat16)
do = torch.randn(S, HQ, D, device="cuda", dtype=torch.bfloat16)
out, lse = ffa_forward(plan, q, k, v)
ffa_backward(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()
print("ok")
