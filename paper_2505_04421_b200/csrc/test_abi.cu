// Test hooks (not part of include/longer.h): single product kernels behind a C entry point, so the
// GPU tests can check them in isolation (tests/test_gemm_gpu.py, tests/test_kat_device_gpu.py).
#include "gemm.cuh"
#include "ops.cuh"

extern "C" int longer_test_gemm(const void* A, int lda, int amn, const void* B, int ldb, int bmn,
                                float* C, int M, int N, int K, int split, void* stream) {
  longer::refresh_knobs();
  longer::GemmArgs g; g.A=A; g.lda=lda; g.a_mn_major=amn; g.B=B; g.ldb=ldb; g.b_mn_major=bmn;
  g.M=M; g.N=N; g.K=K; g.split_k=split; g.flags = longer::EPI_OUT_F32 | (split>1? longer::EPI_ATOMIC:0);
  g.C=C; g.ldc=N;
  return longer::gemm_launch(g, (cudaStream_t)stream);
}

// layernorm_fwd (the query-row / K/V-row LayerNorm of the blocks) over rows x [rows, W] fp32
extern "C" int longer_test_layernorm(const float* x, int rows, int W, const float* g, const float* b, void* y_bf16,
                                     float* mean, float* rstd, void* stream) {
  longer::refresh_knobs();
  longer::RowMap r{};
  r.A = x; r.lda = W; r.a_rows = rows; r.a_off = 0; r.na = rows; r.Bsrc = nullptr; r.ldb = 0; r.nb = 0; r.batch = 1;
  longer::layernorm_fwd(r, W, g, b, reinterpret_cast<longer::bf16*>(y_bf16), mean, rstd, (cudaStream_t)stream);
  return (int)cudaGetLastError();
}
