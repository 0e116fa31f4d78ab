"""Pins the tcgen05/TMA building blocks (descriptor encodings, TMEM layout)
against a torch fp32 matmul of the same bf16 tile."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("b_mn_major", [0, 1, 2])
def test_umma_tile(built_lib, cuda, b_mn_major):
    from paper_2505_13211_b200 import _lib

    g = torch.Generator(device="cpu").manual_seed(0)
    a = torch.randn(128, 128, generator=g).to(torch.bfloat16).to(cuda)
    b = torch.randn(128, 128, generator=g).to(torch.bfloat16).to(cuda)
    c = torch.zeros(128, 128, dtype=torch.float32, device=cuda)
    _lib.call("magiplan_debug_umma_tile", a.data_ptr(), b.data_ptr(), c.data_ptr(), b_mn_major,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = a.float() @ (b.float() if b_mn_major == 1 else b.float().t())
    err = (c - ref).abs().max().item()
    assert err < 1e-3, f"max abs err {err}"
