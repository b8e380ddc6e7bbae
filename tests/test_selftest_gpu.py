"""tcgen05 / TMA / TMEM building-block self test against a torch fp32 GEMM."""
import ctypes

import pytest
import torch

from paper_2503_14376_b200 import _ffi


@pytest.mark.gpu
@pytest.mark.parametrize("a_mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("b_mode", [0, 1])
@pytest.mark.parametrize("N,K", [(64, 64), (128, 128), (256, 256), (128, 256)])
def test_selftest_gemm(a_mode, b_mode, N, K):
    torch.manual_seed(a_mode * 100 + b_mode * 10 + N + K)
    dev = "cuda"
    A = torch.randn(128, K, device=dev).to(torch.bfloat16)  # logical A [128][K]
    B = torch.randn(N, K, device=dev).to(torch.bfloat16)  # logical B [N][K]
    a_arg = A.contiguous() if a_mode in (0, 2, 4) else A.t().contiguous()
    b_arg = B.contiguous() if b_mode == 0 else B.t().contiguous()
    out = torch.zeros(128, N, device=dev, dtype=torch.float32)
    out16 = torch.zeros(128, N, device=dev, dtype=torch.bfloat16)
    rc = _ffi.lib().tfla_selftest_gemm(
        a_mode, b_mode, N, K, a_arg.data_ptr(), b_arg.data_ptr(), out.data_ptr(),
        out16.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
    )
    assert rc == 0, _ffi.last_error()
    torch.cuda.synchronize()
    ref = A.float() @ B.float().t()
    err = (out - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, ref.abs().max().item()), f"max err {err}"
    err16 = (out16.float() - ref).abs().max().item()
    assert err16 < 1e-2 * ref.abs().max().item(), f"bf16 store err {err16}"
