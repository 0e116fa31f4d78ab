"""FFA kernels beside the attention kernels that ship in this image, on masks
every library can express (causal, and block-diagonal documents), at the
headline head layout (24 q heads / 8 kv heads, d = 128, bf16).

Arms (each timed with CUDA events, median of `reps` after warm-up, kernels only):
  ffa          this repo (C ABI via paper_2505_13211_b200.ffa)
  sdpa_cudnn   torch.nn.functional.scaled_dot_product_attention, cuDNN backend
  sdpa_flash   the same, torch's FlashAttention-2 backend
  fi_cutlass   flashinfer.prefill.fmha_varlen (CUTLASS sm100 FMHA; forward
               only, JIT-compiled on first use — skipped when the build fails)

Mask-aware FLOPs as bench.py (fwd 4*area*hq*d, bwd 2.5x). One JSON line per
(mask, arm). Library kernels are comparison points only; nothing on the
product path calls them.

    python tools/compare_attention_libs.py [reps]
"""
from __future__ import annotations

import json
import math
import statistics
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_13211_b200.ffa import FFAPlan, ffa_backward, ffa_forward  # noqa: E402

HQ, HK, D = 24, 8, 128


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def masks():
    S = 32768
    yield "causal S=32768", S, 1, S, True
    yield "8 docs x 4096 full", S, 8, 4096, False
    yield "8 docs x 4096 causal", S, 8, 4096, True


def main(reps: int = 10) -> None:
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    for name, S, ndoc, L, causal in masks():
        q = torch.randn(S, HQ, D, device=dev, generator=g).to(torch.bfloat16)
        k = torch.randn(S, HK, D, device=dev, generator=g).to(torch.bfloat16)
        v = torch.randn(S, HK, D, device=dev, generator=g).to(torch.bfloat16)
        do = torch.randn(S, HQ, D, device=dev, generator=g).to(torch.bfloat16)
        area = ndoc * (L * (L + 1) // 2 if causal else L * L)
        fwd_flops = 4 * area * HQ * D
        rows = []

        # ---- ffa
        plan = FFAPlan([[i * L, (i + 1) * L] for i in range(ndoc)], [[i * L, (i + 1) * L] for i in range(ndoc)],
                       ["causal" if causal else "full"] * ndoc, S, S, D)
        out, lse = ffa_forward(plan, q, k, v)
        t_f = timed(lambda: ffa_forward(plan, q, k, v), reps)
        t_b = timed(lambda: ffa_backward(plan, q, k, v, out, lse, do), reps)
        rows.append(("ffa", t_f, t_b))

        # ---- torch SDPA ([B, H, L, D] views of the same tensors)
        def bhsd(t):
            return t.view(ndoc, L, t.shape[1], D).transpose(1, 2)

        for arm, backend in (("sdpa_cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION),
                             ("sdpa_flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION)):
            try:
                with torch.nn.attention.sdpa_kernel([backend]):
                    qq = bhsd(q).detach().requires_grad_()
                    kk, vv = bhsd(k).detach().requires_grad_(), bhsd(v).detach().requires_grad_()
                    dd = bhsd(do)

                    def fwd():
                        return F.scaled_dot_product_attention(qq, kk, vv, is_causal=causal, enable_gqa=True)

                    t_f = timed(lambda: fwd(), reps)
                    o = fwd()

                    def bwd():
                        torch.autograd.grad(o, (qq, kk, vv), dd, retain_graph=True)

                    t_b = timed(bwd, reps)
                rows.append((arm, t_f, t_b))
            except Exception as e:  # backend not available for this shape / arch
                print(json.dumps({"mask": name, "arm": arm, "unavailable": str(e).splitlines()[0][:200]}))

        # ---- flashinfer CUTLASS sm100 FMHA (forward only)
        try:
            import flashinfer.prefill as fp

            offs = torch.arange(0, S + 1, L, device=dev, dtype=torch.int32)
            out_fi = fp.fmha_varlen(q, k, v, offs, offs, max_qo_len=L, causal=causal, sm_scale=1 / math.sqrt(D))
            if isinstance(out_fi, tuple):
                out_fi = out_fi[0]
            ref = ffa_forward(plan, q, k, v)[0]
            err = float((out_fi.float() - ref.float()).abs().max())
            t_f = timed(lambda: fp.fmha_varlen(q, k, v, offs, offs, max_qo_len=L, causal=causal,
                                               sm_scale=1 / math.sqrt(D)), reps)
            rows.append(("fi_cutlass", t_f, None))
            print(json.dumps({"mask": name, "arm": "fi_cutlass", "max_abs_diff_vs_ffa": round(err, 4)}))
        except Exception as e:
            print(json.dumps({"mask": name, "arm": "fi_cutlass", "unavailable": str(e).splitlines()[0][:200]}))

        for arm, t_f, t_b in rows:
            rec = {"mask": name, "arm": arm, "heads": f"{HQ}q/{HK}kv", "d": D,
                   "fwd_ms": round(t_f, 3), "fwd_tflops": round(fwd_flops / t_f / 1e9, 1)}
            if t_b is not None:
                rec.update(bwd_ms=round(t_b, 3), bwd_tflops=round(2.5 * fwd_flops / t_b / 1e9, 1),
                           fwd_bwd_tflops=round(3.5 * fwd_flops / (t_f + t_b) / 1e9, 1))
            print(json.dumps(rec))
        sys.stdout.flush()
        del q, k, v, do
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10)
