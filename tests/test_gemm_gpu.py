"""tcgen05 GEMM unit test: every operand-major combination against a torch fp32 reference."""
import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2505_04421_b200 import _lib
    return _lib.load()


@pytest.mark.parametrize("amn", [0, 1])
@pytest.mark.parametrize("bmn", [0, 1])
@pytest.mark.parametrize("M,N,K,split", [(128, 64, 64, 1), (304, 256, 200, 1), (8960, 128, 512, 1),
                                         (128, 256, 20000, 8), (77, 96, 136, 1), (8960, 384, 128, 1)])
def test_gemm_matches_torch(amn, bmn, M, N, K, split):
    if (amn and M % 8) or (bmn and N % 8):
        pytest.skip("TMA needs 16-byte row strides")
    lib = _lib()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(K, N, device="cuda", generator=g).bfloat16()
    Ast = A.t().contiguous() if amn else A.contiguous()      # MN-major A stored [K][M]
    Bst = B.contiguous() if bmn else B.t().contiguous()      # MN-major B stored [K][N]
    lda = M if amn else K
    ldb = N if bmn else K
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    rc = lib.longer_test_gemm(ctypes.c_void_p(Ast.data_ptr()), lda, amn, ctypes.c_void_p(Bst.data_ptr()), ldb, bmn,
                              ctypes.c_void_p(C.data_ptr()), M, N, K, split,
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ref = A.float() @ B.float()
    err = (C - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err
