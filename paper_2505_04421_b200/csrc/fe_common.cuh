// fe_common.cuh — shared pieces of the fused front-end kernels (frontend.cu).
//
// Canonical no-swizzle layout (tcgen05 "interleave"): a [rows x Kdim] bf16 tile is stored as 8x8
// core matrices (8 rows x 16 bytes); element (row, k) lives at canon(row, k, Kdim).  The same bytes
// serve as a K-major operand (rows = M/N, LBO = 128 B, SBO = Kdim*16 B) or, for weight-gradient
// MMAs that contract over the 128 token rows, as an MN-major operand (LBO = Kdim*16 B, SBO = 128 B).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "sm100.cuh"

namespace longer {
namespace fe {

constexpr int kFP = 32;                 // featuriser K: F = d_item + d_act + d_time padded to 32
constexpr int kTile = 128;              // tokens per tile (= UMMA M = TMEM lanes)
constexpr int kWorkers = 4;
constexpr int kThreads = 32 * (1 + kWorkers);
constexpr int kThreads8 = 32 * (1 + 2 * kWorkers);   // MMA warp + 8 worker warps (two per lane quarter)

__host__ __device__ __forceinline__ int canon(int row, int k, int Kdim) {
  return (row >> 3) * (Kdim * 8) + (k >> 3) * 64 + (row & 7) * 8 + (k & 7);
}

// element offsets of every weight image inside the packed blob (forward images WxT = [out][in],
// backward images Wx_n = [in][out], both canonical K-major).  Forward images whose activation
// tile carries a ones column get one extra K row holding the bias ("bias-augmented", K = d + 16,
// bias at k = d; for W_tp the bias sits in the spare feature column k = 31), so those biases are
// added by the tensor core instead of the epilogue.
struct BlobOff {
  int tp, w1, w2;                       // forward: [Wtpᵀ|b] [d][32], [W1ᵀ|b1] [2D][d+16], W2ᵀ [d][2D]
  int tp_n, w1_n, w2_n;                 // backward: Wtp [32][d], W1 [d][2D], W2 [2D][d]
  int qkv[8], wo[8], w1i[8], w2i[8];    // forward inner: [3d][d+16], [d][d], [4d][d+16], [d][4d]
  int qkv_n[8], wo_n[8], w1i_n[8], w2i_n[8];  // backward inner: [d][3d], [d][d], [d][4d], [4d][d]
  int fwd_total, total;
};

__host__ __device__ inline BlobOff blob_offsets(int d, int D, int IL) {
  BlobOff o;
  int off = 0;
  const int XK = d + 16;
  o.tp = off; off += d * kFP;
  o.w1 = off; off += 2 * D * XK;
  o.w2 = off; off += d * 2 * D;
  for (int l = 0; l < IL; ++l) {
    o.qkv[l] = off; off += 3 * d * XK;
    o.wo[l] = off; off += d * d;
    o.w1i[l] = off; off += 4 * d * XK;
    o.w2i[l] = off; off += d * 4 * d;
  }
  o.fwd_total = off;
  o.tp_n = off; off += kFP * d;
  o.w1_n = off; off += d * 2 * D;
  o.w2_n = off; off += 2 * D * d;
  for (int l = 0; l < IL; ++l) {
    o.qkv_n[l] = off; off += d * 3 * d;
    o.wo_n[l] = off; off += d * d;
    o.w1i_n[l] = off; off += d * 4 * d;
    o.w2i_n[l] = off; off += 4 * d * d;
  }
  o.total = off;
  return o;
}

__device__ __forceinline__ void store_row(bf16* tile, int row, int Kdim, const float* v, int n, int k0 = 0) {
#pragma unroll
  for (int c = 0; c < n; c += 8) {
    uint4 pk;
    pk.x = sm100::pack_bf16(v[c + 0], v[c + 1]);
    pk.y = sm100::pack_bf16(v[c + 2], v[c + 3]);
    pk.z = sm100::pack_bf16(v[c + 4], v[c + 5]);
    pk.w = sm100::pack_bf16(v[c + 6], v[c + 7]);
    *reinterpret_cast<uint4*>(tile + canon(row, k0 + c, Kdim)) = pk;
  }
}

// Operand view of a canonical tile.  mn = 0: K-major (tile rows = M/N); mn = 1: MN-major (tile
// rows = the K dimension, i.e. the 128 tokens of a weight-gradient contraction).
struct Opnd {
  uint32_t addr;
  int kdim;     // the tile's row length in elements
  int mn;
  __device__ __forceinline__ uint64_t desc(int ks) const {
    return mn ? sm100::make_sdesc(addr + ks * 2 * (kdim * 16), kdim * 16, 128, sm100::LAYOUT_NONE)
              : sm100::make_sdesc(addr + ks * 256, 128, kdim * 16, sm100::LAYOUT_NONE);
  }
};

// Operand view of a [rows][64·nb] tile written by TMA as nb column blocks of 64 (128-byte swizzle,
// block stride rows·128 bytes).  mn = 0: K-major (contraction over the columns, N = rows);
// mn = 1: MN-major (contraction over the rows, N = the columns).
struct OpndSW {
  uint32_t addr;
  int rows;
  int mn;
  __device__ __forceinline__ uint64_t desc(int ks) const {
    return mn ? sm100::make_sdesc(addr + ks * 2048, rows * 128, 1024, sm100::LAYOUT_SW128)
              : sm100::make_sdesc(addr + (ks >> 2) * rows * 128 + (ks & 3) * 32, 16, 1024, sm100::LAYOUT_SW128);
  }
};

// D[tmem, 128 x N] (+)= A · B over `kslices` K-slices of 16 (single thread)
template <class OA, class OB>
__device__ __forceinline__ void mma(uint32_t tmem_d, const OA& A, const OB& B, int kslices, int N, bool acc) {
  const uint32_t idesc = sm100::make_idesc_bf16(128, N, A.mn, B.mn);
  for (int ks = 0; ks < kslices; ++ks)
    sm100::mma_bf16(tmem_d, A.desc(ks), B.desc(ks), idesc, (acc || ks > 0) ? 1u : 0u);
}

// issue the loads of N columns (N = 16 or a multiple of 32) without waiting
template <int N>
__device__ __forceinline__ void tmem_row_issue(uint32_t taddr, uint32_t* r) {
#pragma unroll
  for (int c = 0; c < N; c += 32) {
    if (c + 32 <= N) sm100::tmem_ld32(taddr + c, *reinterpret_cast<uint32_t(*)[32]>(r + c));
    else sm100::tmem_ld16(taddr + c, *reinterpret_cast<uint32_t(*)[16]>(r + c));
  }
}
// after tcgen05.wait::ld: tie each loaded register to the wait, so no use is scheduled above it
template <int N>
__device__ __forceinline__ void tmem_row_take(uint32_t* r, float* out) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    asm volatile("" : "+r"(r[j]));
    out[j] = __uint_as_float(r[j]);
  }
}
// one row's N TMEM columns → out (all loads in flight together, one wait)
template <int N>
__device__ __forceinline__ void tmem_row(uint32_t taddr, float* out) {
  uint32_t r[N];
  tmem_row_issue<N>(taddr, r);
  sm100::tmem_ld_wait();
  tmem_row_take<N>(r, out);
}
// two rows of columns (e.g. an accumulator and its gradient) with one wait
template <int N>
__device__ __forceinline__ void tmem_row2(uint32_t ta, float* a, uint32_t tb, float* b) {
  uint32_t ra[N], rb[N];
  tmem_row_issue<N>(ta, ra);
  tmem_row_issue<N>(tb, rb);
  sm100::tmem_ld_wait();
  tmem_row_take<N>(ra, a);
  tmem_row_take<N>(rb, b);
}

// park a row's N fp32 values in TMEM columns [taddr, taddr + N) (N = 16 or a multiple of 32)
template <int N>
__device__ __forceinline__ void tmem_row_st(uint32_t taddr, const float* v) {
#pragma unroll
  for (int c = 0; c < N; c += 32) {
    if (c + 32 <= N) {
      uint32_t r[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(v[c + j]);
      sm100::tmem_st32(taddr + c, r);
    } else {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(v[c + j]);
      sm100::tmem_st16(taddr + c, r);
    }
  }
  sm100::tmem_st_wait();
}

template <int DT>
__device__ __forceinline__ void ln_row(const float* x, const float* g, const float* b, float* y, float* xhat,
                                       float& inv_out) {
  float mu = 0.f;
#pragma unroll
  for (int c = 0; c < DT; ++c) mu += x[c];
  mu *= 1.f / DT;
  float var = 0.f;
#pragma unroll
  for (int c = 0; c < DT; ++c) { const float t = x[c] - mu; var += t * t; }
  const float inv = rsqrtf(var * (1.f / DT) + kLnEps);
  inv_out = inv;
#pragma unroll
  for (int c = 0; c < DT; ++c) {
    const float xh = (x[c] - mu) * inv;
    if (xhat) xhat[c] = xh;
    y[c] = xh * __ldg(g + c) + __ldg(b + c);
  }
}

// Column sums of a warp's 32 rows: on return lane c holds Σ_rows v[c] (c < W; W ∈ {16, 32}).
// Recursive halving, 31 shuffles for W = 32.
// ln_row with the gain / bias vectors in shared memory (plain loads; ln_row uses the read-only path)
template <int DT>
__device__ __forceinline__ void ln_row_s(const float* x, const float* g, const float* b, float* y, float& inv_out) {
  float mu = 0.f;
#pragma unroll
  for (int c = 0; c < DT; ++c) mu += x[c];
  mu *= 1.f / DT;
  float var = 0.f;
#pragma unroll
  for (int c = 0; c < DT; ++c) { const float t = x[c] - mu; var += t * t; }
  const float inv = rsqrtf(var * (1.f / DT) + kLnEps);
  inv_out = inv;
#pragma unroll
  for (int c = 0; c < DT; ++c) y[c] = (x[c] - mu) * inv * g[c] + b[c];
}

template <int W>
__device__ __forceinline__ float warp_colsum(float (&v)[W]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = W / 2; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float mine = up ? v[w + i] : v[i];
      const float theirs = up ? v[i] : v[w + i];
      v[i] = mine + __shfl_xor_sync(0xffffffffu, theirs, w);
    }
  }
  float r = v[0];
  if (W == 16) r += __shfl_xor_sync(0xffffffffu, r, 16);
  return r;   // column (lane % W)
}

}  // namespace fe
}  // namespace longer
