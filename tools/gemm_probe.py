"""Time the generic tcgen05 GEMM on representative shapes (CUDA events) — profiling helper."""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_04421_b200 import _lib  # noqa: E402

lib = _lib.load()
shapes = [(8960, 512, 128, 0, 1), (8960, 128, 128, 0, 1), (8960, 128, 512, 0, 1), (128768, 256, 128, 0, 1),
          (128768, 128, 256, 0, 0), (128, 256, 128768, 1, 1)]
for M, N, K, amn, bmn in shapes:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    Ast = A.t().contiguous() if amn else A
    Bst = B if bmn else B.t().contiguous()
    C = torch.zeros(M, N, device="cuda")
    split = 0 if amn else 1
    args = (ctypes.c_void_p(Ast.data_ptr()), M if amn else K, amn, ctypes.c_void_p(Bst.data_ptr()), N if bmn else K,
            bmn, ctypes.c_void_p(C.data_ptr()), M, N, K, 148 if amn else 1,
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        assert lib.longer_test_gemm(*args) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lib.longer_test_gemm(*args)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
    gb = (M * K * 2 + K * N * 2 + M * N * 4) / (us * 1e-6) / 1e9
    print(f"M={M} N={N} K={K} amn={amn}: {us:8.1f} us  {tf:7.1f} TFLOP/s  {gb:7.0f} GB/s")
