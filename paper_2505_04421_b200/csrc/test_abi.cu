#include "gemm.cuh"
extern "C" int longer_test_gemm(const void* A, int lda, int amn, const void* B, int ldb, int bmn,
                                float* C, int M, int N, int K, int split, void* stream) {
  longer::GemmArgs g; g.A=A; g.lda=lda; g.a_mn_major=amn; g.B=B; g.ldb=ldb; g.b_mn_major=bmn;
  g.M=M; g.N=N; g.K=K; g.split_k=split; g.flags = longer::EPI_OUT_F32 | (split>1? longer::EPI_ATOMIC:0);
  g.C=C; g.ldc=N;
  return longer::gemm_launch(g, (cudaStream_t)stream);
}
