"""Time one GEMM shape of the generic tcgen05 GEMM (CUDA events) — profiling helper.
Usage: python tools/gemm_one.py M N K [amn bmn] [iters]"""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_04421_b200 import _lib  # noqa: E402

lib = _lib.load()
M, N, K = (int(v) for v in sys.argv[1:4])
amn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
bmn = int(sys.argv[5]) if len(sys.argv) > 5 else 1
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 10
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(K, N, device="cuda").bfloat16()
Ast = A.t().contiguous() if amn else A
Bst = B if bmn else B.t().contiguous()
C = torch.zeros(M, N, device="cuda")
args = (ctypes.c_void_p(Ast.data_ptr()), M if amn else K, amn, ctypes.c_void_p(Bst.data_ptr()), N if bmn else K,
        bmn, ctypes.c_void_p(C.data_ptr()), M, N, K, 148 if amn else 1,
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
for _ in range(3):
    assert lib.longer_test_gemm(*args) == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    lib.longer_test_gemm(*args)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / iters
ref = (A.float() @ B.float())
err = (C - ref).abs().max().item() / ref.abs().max().item()
gb = (M * K * 2 + K * N * 2 + M * N * 4) / (us * 1e-6) / 1e9
print(f"M={M} N={N} K={K} amn={amn} bmn={bmn}: {us:8.1f} us  {2.0 * M * N * K / (us * 1e-6) / 1e12:7.1f} TFLOP/s"
      f"  {gb:7.0f} GB/s  rel_err {err:.2e}")
