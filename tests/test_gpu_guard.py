"""Out-of-bounds guard: every output of the forward / backward C ABI calls is
carved out of a larger buffer filled with a canary pattern, at sizes that are
not multiples of the 128-row tiles. The kernels must write exactly their
outputs (every canary byte outside them intact) and leave the inputs
unchanged. (compute-sanitizer is not available on the GPU pool; this is the
bounds check of our own.)
"""
import math

import pytest
import torch

from tests.ffa_cases import CASES, make_inputs

pytestmark = pytest.mark.gpu

PAD = 64 * 1024  # canary bytes on each side of every output
CANARY = 0x5A


def _guarded(numel, dtype, dev):
    """A view of `numel` elements in the middle of a canary-filled byte buffer."""
    esize = torch.empty((), dtype=dtype).element_size()
    raw = torch.full((2 * PAD + numel * esize,), CANARY, dtype=torch.uint8, device=dev)
    view = raw[PAD:PAD + numel * esize].view(dtype)
    return raw, view


def _canaries_intact(raw, numel_bytes):
    return bool((raw[:PAD] == CANARY).all()) and bool((raw[PAD + numel_bytes:] == CANARY).all())


@pytest.mark.parametrize("name", ["causal_unaligned", "many_tiny_docs", "cross_lk_gt_lq", "gqa6_causal_d64",
                                  "uncovered_keys"])
@pytest.mark.parametrize("grad_f32", [False, True])
def test_outputs_stay_in_bounds(built_lib, cuda, name, grad_f32):
    from paper_2505_13211_b200 import _lib
    from paper_2505_13211_b200.ffa import FFAPlan

    sq, sk, hq, hk, d, qr, kr, ty = CASES[name]
    dev = torch.device("cuda", 0)
    q, k, v, do = make_inputs(sq, sk, hq, hk, d, seed=3)
    inputs = [t.clone() for t in (q, k, v, do)]
    plan = FFAPlan(qr, kr, ty, sq, sk, d)
    L, BF, F32 = _lib.lib(), _lib.BF16, _lib.F32
    gdt = torch.float32 if grad_f32 else torch.bfloat16
    bufs = {
        "out": _guarded(sq * hq * d, torch.bfloat16, dev),
        "lse": _guarded(hq * sq, torch.float32, dev),
        "delta": _guarded(hq * sq, torch.float32, dev),
        "dq": _guarded(sq * hq * d, gdt, dev),
        "dk": _guarded(sk * hk * d, gdt, dev),
        "dv": _guarded(sk * hk * d, gdt, dev),
    }
    p = {n: b[1].data_ptr() for n, b in bufs.items()}
    sp = torch.cuda.current_stream(dev).cuda_stream
    scale = 1.0 / math.sqrt(d)
    _lib.check(L.magiplan_ffa_fwd(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), p["out"], p["lse"],
                                  hq, hk, scale, BF, 0, sp))
    _lib.check(L.magiplan_ffa_bwd_preprocess(p["out"], do.data_ptr(), p["delta"], sq, hq, d, BF, sp))
    _lib.check(L.magiplan_ffa_bwd(plan.handle, q.data_ptr(), k.data_ptr(), v.data_ptr(), p["lse"], p["delta"],
                                  do.data_ptr(), p["dq"], p["dk"], p["dv"], hq, hk, scale,
                                  F32 if grad_f32 else BF, 0, sp))
    torch.cuda.synchronize()
    for n, (raw, view) in bufs.items():
        assert _canaries_intact(raw, view.numel() * view.element_size()), f"{name}: write outside {n}"
    for a, b in zip(inputs, (q, k, v, do)):
        assert torch.equal(a, b), f"{name}: an input was modified"


def test_range_ops_stay_in_bounds(built_lib, cuda):
    """Range Gather / Scatter-Reduce with ragged ranges (lengths 1..37 rows,
    one empty) write only their packed / scattered rows, and match a torch
    restatement exactly."""
    from paper_2505_13211_b200 import _lib

    dev = torch.device("cuda", 0)
    L = _lib.lib()
    sp = torch.cuda.current_stream(dev).cuda_stream
    rows, width = 300, 48  # f32 row = 192 B
    g = torch.Generator(device="cpu").manual_seed(5)
    src = torch.randn(rows, width, generator=g).to(dev)
    bounds = [(3, 40), (40, 41), (77, 77), (100, 137), (250, 300), (0, 2)]
    total = sum(e - s for s, e in bounds)
    offs, o = [], 0
    for s, e in bounds:
        offs.append(o)
        o += e - s
    ranges = torch.tensor(bounds, dtype=torch.int64, device=dev)
    offsets = torch.tensor(offs, dtype=torch.int64, device=dev)
    raw, dst = _guarded(total * width, torch.float32, dev)
    _lib.check(L.magiplan_range_gather(src.data_ptr(), dst.data_ptr(), ranges.data_ptr(), offsets.data_ptr(),
                                       len(bounds), total, width * 4, sp))
    torch.cuda.synchronize()
    assert _canaries_intact(raw, total * width * 4)
    want = torch.cat([src[s:e] for s, e in bounds])
    assert torch.equal(dst.view(total, width), want)
    # scatter-add the packed rows back onto a guarded accumulator
    raw2, acc = _guarded(rows * width, torch.float32, dev)
    acc.zero_()
    _lib.check(L.magiplan_range_scatter_add_f32(dst.data_ptr(), acc.data_ptr(), ranges.data_ptr(),
                                                offsets.data_ptr(), len(bounds), total, width, sp))
    torch.cuda.synchronize()
    assert _canaries_intact(raw2, rows * width * 4)
    ref = torch.zeros(rows, width, device=dev)
    for (s, e), off in zip(bounds, offs):
        ref[s:e] += want[off:off + e - s]
    assert torch.equal(acc.view(rows, width), ref)
