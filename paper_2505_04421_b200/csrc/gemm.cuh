// gemm.cuh — generic warp-specialised tcgen05 GEMM with fused epilogues (sm_100a).
//
//   C[M,N] = epi( A[M,K] · B[K,N] )      bf16 operands, fp32 accumulation in TMEM
//
// Operand majors:  A K-major = row-major [M][K];  A MN-major = stored [K][M]
//                  B K-major = stored [N][K];     B MN-major = row-major [K][N]
// so Y = X·W (W stored [in,out]) is (A K-major, B MN-major); dX = dY·Wᵀ is (K, K);
// dW = Xᵀ·dY is (A MN-major, B MN-major).  Tiles: BM=128, BN∈{64,128,256}, BK=64,
// 4-stage TMA→smem ring (128B swizzle), one MMA thread, 4 epilogue warps (row = TMEM lane).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace longer {

enum EpiFlags : uint32_t {
  EPI_BIAS = 1u << 0,       // + bias[n]                     (fp32)
  EPI_GELU = 1u << 1,       // tanh-GELU after bias
  EPI_RESID = 1u << 2,      // + resid[m, n] (fp32, ld = ldr) after activation
  EPI_OUT_F32 = 1u << 3,    // write fp32 C (ldc)
  EPI_OUT_BF16 = 1u << 4,   // write bf16 copy (ldc_bf)
  EPI_ATOMIC = 1u << 5,     // fp32 atomicAdd into C (split-K / gradient accumulation)
  EPI_SAVE_PRE = 1u << 6,   // store pre-activation (bf16, ld = ldc_bf) into pre_bf16
  EPI_ROWMASK = 1u << 7,    // multiply output rows by rowmask[m] (0/1 fp32)
  EPI_GELU_BWD = 1u << 8,   // multiply by GELU'(pre[m, n]) (pre_bf16 is an INPUT, ld = ldc_bf)
};

struct GemmArgs {
  const void* A = nullptr; int lda = 0; int a_mn_major = 0;   // bf16
  const void* B = nullptr; int ldb = 0; int b_mn_major = 0;   // bf16
  int M = 0, N = 0, K = 0;
  int split_k = 1;                  // >1 → K split across gridDim.z (requires EPI_ATOMIC); 0 = auto
  uint32_t flags = EPI_OUT_F32;
  const float* bias = nullptr;
  const float* resid = nullptr; int ldr = 0;
  const float* rowmask = nullptr;
  float* C = nullptr; int ldc = 0;
  void* C_bf16 = nullptr; int ldc_bf = 0;
  void* pre_bf16 = nullptr;         // pre-activation out (EPI_SAVE_PRE), ld = ldc_bf
  int staged = -1;                  // epilogue stores through a per-warp smem transpose (-1: LONGER_GEMM_STAGE)
  int late_trigger = 0;             // set by the launcher (LONGER_GEMM_LATE_TRIGGER)
};

// Host: encodes the TMA descriptors and launches. Returns a cudaError_t value (0 = ok).
int gemm_launch(const GemmArgs& g, cudaStream_t stream);

}  // namespace longer
