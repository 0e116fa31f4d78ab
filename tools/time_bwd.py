"""Development timing of the FFA passes for one build of the library:

    python tools/time_bwd.py [path/to/libmagiplan.so] [workload]

workload: a bench.py WORKLOADS key (default config 2: S = 32768, block-causal
4096, 24 q / 8 kv heads, d = 128). Prints ms per call of the forward, the
whole backward (dQ, dK, dV), the dK/dV pass and the dQ pass."""
import json
import math
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_13211_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib._LIB_PATH = Path(sys.argv[1]).resolve()
import bench  # noqa: E402
from paper_2505_13211_b200.ffa import FFAPlan  # noqa: E402

WL = sys.argv[2] if len(sys.argv) > 2 else bench.DEFAULT_WORKLOAD
W = bench.WORKLOADS[WL]
S, HQ, HK, D, B = W["seqlen"], W["hq"], W["hk"], W["d"], W["block"]
if W.get("varlen"):
    qr, kr, ty = bench.varlen_packed(S)
else:
    qr = [[i, i + B] for i in range(0, S, B)]
    kr = [[0, i + B] for i in range(0, S, B)]
    ty = [0] * len(qr)
plan = FFAPlan(qr, kr, ty, S, S, D)
dev = torch.device("cuda", 0)
q = torch.randn(S, HQ, D, device=dev, dtype=torch.bfloat16)
k = torch.randn(S, HK, D, device=dev, dtype=torch.bfloat16)
v = torch.randn(S, HK, D, device=dev, dtype=torch.bfloat16)
do = torch.randn(S, HQ, D, device=dev, dtype=torch.bfloat16)
out = torch.empty_like(q)
lse = torch.empty(HQ, S, device=dev)
delta = torch.empty(HQ, S, device=dev)
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
L = _lib.lib()
sp = torch.cuda.current_stream(dev).cuda_stream
sc = 1 / math.sqrt(D)
BF = _lib.BF16
fwd = lambda: _lib.check(L.magiplan_ffa_fwd(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),  # noqa: E731
                                            lse.data_ptr(), HQ, HK, sc, BF, 0, sp))
fwd()
_lib.check(L.magiplan_ffa_bwd_preprocess(out.data_ptr(), do.data_ptr(), delta.data_ptr(), S, HQ, D, BF, sp))
bwd = lambda: _lib.check(L.magiplan_ffa_bwd(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), lse.data_ptr(),  # noqa: E731
                                            delta.data_ptr(), do.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                                            dv.data_ptr(), HQ, HK, sc, BF, 0, sp))
dkdv = lambda: _lib.check(L.magiplan_ffa_bwd_dkdv(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),  # noqa: E731
                                                  lse.data_ptr(), delta.data_ptr(), do.data_ptr(), dk.data_ptr(),
                                                  dv.data_ptr(), HQ, HK, sc, BF, 0, sp))


def t(fn, n=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


area = plan.describe()["area_multiplicity"]
dqo = lambda: _lib.check(L.magiplan_ffa_bwd_dq(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(),  # noqa: E731
                                                lse.data_ptr(), delta.data_ptr(), do.data_ptr(), dq.data_ptr(),
                                                HQ, HK, sc, BF, 0, sp))
res = {"lib": str(_lib._LIB_PATH), "workload": WL, "fwd_ms": t(fwd), "bwd_ms": t(bwd), "dkdv_only_ms": t(dkdv),
       "dq_only_ms": t(dqo)}
res["fwd_tflops"] = 4 * area * HQ * D / res["fwd_ms"] / 1e9
res["bwd_tflops"] = 10 * area * HQ * D / res["bwd_ms"] / 1e9
print(json.dumps(res))
