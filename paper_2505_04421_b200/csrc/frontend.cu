// frontend.cu — fused token front-end, forward (see frontend.cuh).
//
// Restates, per token: _event_features + abs-pos (pkg/src/longrec/inputs.py:434-482), the token
// MLP (inputs.py:447-449), and merge_inner_trans (pkg/src/longrec/merge.py:83-112) with
// grouped_attention (pkg/src/longrec/tensors.py:406-444), for 128-token tiles.
//
// CTA = warp 0 (TMEM owner + single-thread MMA issuer) + 4 worker warps (thread = token row =
// TMEM lane).  Per stage: workers write the A tile (bf16, canonical no-swizzle K-major) → mbarrier
// → one thread issues tcgen05.mma (M=128) against the smem-resident weight blob → tcgen05.commit →
// workers read the fp32 accumulator from TMEM and apply bias / GELU / LN / group attention in
// registers.  Two CTAs per SM overlap one CTA's MMA with the other's epilogue math.
#include "frontend.cuh"
#include "sm100.cuh"

#include <algorithm>

namespace longer {

namespace {

constexpr int kFP = 32;                 // featuriser K (F = d_item + d_act + d_time padded)
constexpr int kTile = 128;
constexpr int kWorkers = 4;
constexpr int kThreads = 32 * (1 + kWorkers);
constexpr int kTmemCols = 256;

// canonical K-major, no swizzle: element (row, k) of a [rows x Kdim] bf16 tile
__host__ __device__ __forceinline__ int canon(int row, int k, int Kdim) {
  return (row >> 3) * (Kdim * 8) + (k >> 3) * 64 + (row & 7) * 8 + (k & 7);
}

struct BlobOff {          // element offsets inside the weight blob
  int tp, w1, w2;
  int qkv[8], wo[8], w1i[8], w2i[8];
  int total;
};

__host__ __device__ inline BlobOff blob_offsets(int d, int D, int IL) {
  BlobOff o;
  int off = 0;
  o.tp = off; off += d * kFP;
  o.w1 = off; off += 2 * D * d;
  o.w2 = off; off += d * 2 * D;
  for (int l = 0; l < IL; ++l) {
    o.qkv[l] = off; off += 3 * d * d;
    o.wo[l] = off; off += d * d;
    o.w1i[l] = off; off += 4 * d * d;
    o.w2i[l] = off; off += d * 4 * d;
  }
  o.total = off;
  return o;
}

// ------------------------------------------------------------------ weight packing
struct PackW {
  int n;
  struct { long long src; int in, out, n_off, Kdim, dst; } s[40];
};

__global__ void pack_canon_kernel(const float* __restrict__ params, PackW pw, bf16* blob) {
  const auto s = pw.s[blockIdx.y];
  const int N = s.out, Kd = s.Kdim;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * Kd; e += gridDim.x * blockDim.x) {
    const int n = e / Kd, k = e % Kd;
    const float v = k < s.in ? params[s.src + (long long)k * s.out + n] : 0.f;
    blob[s.dst + canon(s.n_off + n, k, Kd)] = __float2bfloat16(v);
  }
}

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ void store_row_canon(bf16* tile, int row, int Kdim, const float* v, int n, int k0 = 0) {
  // n is a multiple of 8; 16-byte stores per 8-element chunk (columns k0 .. k0+n)
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

// issue D[tmem] (+)= A[smem, 128 x K] · B[smem, N x K]ᵀ as K/16 MMAs (one thread)
__device__ __forceinline__ void mma_tile(uint32_t tmem_d, uint32_t a_addr, int a_kdim, uint32_t b_addr, int b_kdim,
                                         int kslices, int N, bool accumulate) {
  const uint32_t idesc = sm100::make_idesc_bf16(128, N, 0, 0);
  for (int ks = 0; ks < kslices; ++ks) {
    const uint64_t ad = sm100::make_sdesc(a_addr + ks * 256, 128, a_kdim * 16, sm100::LAYOUT_NONE);
    const uint64_t bd = sm100::make_sdesc(b_addr + ks * 256, 128, b_kdim * 16, sm100::LAYOUT_NONE);
    sm100::mma_bf16(tmem_d, ad, bd, idesc, (accumulate || ks > 0) ? 1u : 0u);
  }
}

template <int N>
__device__ __forceinline__ void tmem_row(uint32_t taddr, float* out) {   // N multiple of 16
#pragma unroll
  for (int c = 0; c < N; c += 32) {
    if (c + 32 <= N) {
      uint32_t r[32];
      sm100::tmem_ld32(taddr + c, r);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) out[c + j] = __uint_as_float(r[j]);
    } else {
      uint32_t r[16];
      sm100::tmem_ld16(taddr + c, r);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) out[c + j] = __uint_as_float(r[j]);
    }
  }
}

template <int DT>
__device__ __forceinline__ void layer_norm_row(const float* x, const float* g, const float* b, float* y) {
  float mu = 0.f;
#pragma unroll
  for (int c = 0; c < DT; ++c) mu += x[c];
  mu *= 1.f / DT;
  float var = 0.f;
#pragma unroll
  for (int c = 0; c < DT; ++c) { const float t = x[c] - mu; var += t * t; }
  const float inv = rsqrtf(var * (1.f / DT) + kLnEps);
#pragma unroll
  for (int c = 0; c < DT; ++c) y[c] = (x[c] - mu) * inv * __ldg(g + c) + __ldg(b + c);
}

// ------------------------------------------------------------------ forward kernel
template <int DT, int KG>
__global__ void __launch_bounds__(kThreads, 2) fe_fwd_kernel(FrontArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int D = DT * KG;
  const int H2 = 2 * D;                        // token-MLP hidden width
  const int nh = H2 / 128;                     // 128-column halves of the hidden
  const BlobOff bo = blob_offsets(DT, D, a.inner_layers);
  bf16* sW = reinterpret_cast<bf16*>(smem_raw);
  bf16* sA = sW + ((bo.total + 63) & ~63);                 // 128 x 32 bf16
  bf16* sH = sA + kTile * kFP;                             // 128 x 128 bf16 (also fp32 k/v scratch)
  float* sKV = reinterpret_cast<float*>(sH);               // 128 x (2*DT+1) fp32
  uint64_t* bars = reinterpret_cast<uint64_t*>(sH + kTile * 136);
  uint64_t* bar_w = bars;
  uint64_t* bar_a = bars + 1;
  uint64_t* bar_d = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_w, 1);
    sm100::mbar_init(bar_a, 32 * kWorkers);
    sm100::mbar_init(bar_d, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const long long ntiles = (a.T + kTile - 1) / kTile;

  if (warp == 0) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const int wbytes = bo.total * 2;
      sm100::mbar_arrive_expect_tx(bar_w, wbytes);
      for (int off = 0; off < wbytes; off += 32768) {
        const int n = min(32768, wbytes - off);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(sm100::smem_u32(reinterpret_cast<uint8_t*>(sW) + off)),
                        "l"(reinterpret_cast<const uint8_t*>(a.wblob) + off), "r"(n), "r"(sm100::smem_u32(bar_w))
                     : "memory");
      }
      sm100::mbar_wait(bar_w, 0);
      const uint32_t wA = sm100::smem_u32(sA), wH = sm100::smem_u32(sH), wW = sm100::smem_u32(sW);
      uint32_t pa = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      const uint32_t accH = tmem + 128;          // h / f2 accumulator columns
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        wait_a();                                // feat ready
        mma_tile(tmem, wA, kFP, wW + bo.tp * 2, kFP, kFP / 16, DT, false);
        sm100::mma_commit(bar_d);
        wait_a();                                // x0 ready
        mma_tile(tmem, wA, DT, wW + bo.w1 * 2, DT, DT / 16, 128, false);
        sm100::mma_commit(bar_d);
        for (int j = 0; j < nh; ++j) {
          wait_a();                              // GELU(a1 half j) in sH
          // h (+)= g1_half_j · W2ᵀ[:, 128j : 128j+128]
          mma_tile(accH, wH, 128, wW + (bo.w2 + canon(0, 128 * j, H2)) * 2, H2, 8, DT, j > 0);
          if (j + 1 < nh) mma_tile(tmem, wA, DT, wW + (bo.w1 + canon(128 * (j + 1), 0, DT)) * 2, DT, DT / 16, 128, false);
          sm100::mma_commit(bar_d);
        }
        for (int l = 0; l < a.inner_layers; ++l) {
          wait_a();                              // LN1(x)
          mma_tile(tmem, wA, DT, wW + bo.qkv[l] * 2, DT, DT / 16, 3 * DT, false);
          sm100::mma_commit(bar_d);
          wait_a();                              // ctx
          mma_tile(tmem, wA, DT, wW + bo.wo[l] * 2, DT, DT / 16, DT, false);
          sm100::mma_commit(bar_d);
          wait_a();                              // LN2(x1)
          mma_tile(tmem, wA, DT, wW + bo.w1i[l] * 2, DT, DT / 16, 4 * DT, false);
          sm100::mma_commit(bar_d);
          wait_a();                              // GELU(f1)
          mma_tile(accH, wH, 4 * DT, wW + bo.w2i[l] * 2, 4 * DT, 4 * DT / 16, DT, false);
          sm100::mma_commit(bar_d);
        }
      }
    }
  } else {
    // ---------------- workers: one token row per thread
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int F = a.d_item + a.d_act + a.d_time;
    const float scale_in = rsqrtf((float)DT);
    uint32_t pd = 0;
    auto signal = [&]() {
      sm100::fence_async_smem();
      sm100::tc_fence_before();
      sm100::mbar_arrive(bar_a);
    };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const long long t = tile * kTile + row;
      const bool in_range = t < a.T;
      int b = 0, j = 0, n = 0;
      if (in_range) { b = (int)(t / a.Lp); j = (int)(t % a.Lp); n = min(max(a.n_events[b], 0), a.L); }
      const bool real = in_range && j >= a.Lp - n;
      const int npg = (a.Lp - n) / a.K;
      const bool keep = in_range && (j / a.K) >= npg;
      if (in_range && j == 0 && a.npg) a.npg[b] = npg;
      // S0: featurise
      float v[kFP];
#pragma unroll
      for (int c = 0; c < kFP; ++c) v[c] = 0.f;
      int rec = 0;
      if (real) {
        const long long src = (long long)b * a.L + (j - (a.Lp - a.L));
        int item = a.items[src], act = a.actions[src], dt = a.dt[src];
        int bad = 0;
        if (item < 0 || item >= a.vocab) { bad |= 1; item = 0; }
        if (act < 0 || act >= a.n_actions) { bad |= 1; act = 0; }
        if (dt < 0) { bad |= 2; dt = 0; }
        if (bad) atomicOr(a.status, bad);
        const int bucket = min(32 - __clz(dt), a.nb - 1);
        rec = a.Lp - 1 - j;
        const int e1 = a.d_item, e2 = a.d_item + a.d_act, e3 = e2 + a.d_time;
#pragma unroll
        for (int c = 0; c < kFP; ++c) {
          const float* src_p = c < e1 ? a.item_tab + item * a.d_item + c
                             : c < e2 ? a.act_tab + act * a.d_act + (c - e1)
                                      : a.time_tab + bucket * a.d_time + (c - e2);
          v[c] = c < e3 ? __ldg(src_p) : 0.f;
        }
      }
      (void)F;
      store_row_canon(sA, row, kFP, v, kFP);
      signal();
      // S1: x0 = feat·W_tp + b_tp + abs_pos[recency]
      float x[DT];
      wait_d();
      tmem_row<DT>(trow, x);
#pragma unroll
      for (int c = 0; c < DT; ++c) x[c] = real ? x[c] + __ldg(a.tok_b + c) + __ldg(a.pos_tab + (long long)rec * DT + c) : 0.f;
      store_row_canon(sA, row, DT, x, DT);
      signal();
      // S2: token MLP, hidden in 128-column halves: GELU(x0·W1 + b1) → sH → (·W2) accumulates in TMEM
      for (int hj = 0; hj < nh; ++hj) {
        wait_d();
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          float hv[32];
          tmem_row<32>(trow + c0, hv);
#pragma unroll
          for (int u = 0; u < 32; ++u) hv[u] = gelu_f(hv[u] + __ldg(a.seq_b1 + 128 * hj + c0 + u));
          store_row_canon(sH, row, 128, hv, 32, c0);
        }
        signal();
      }
      wait_d();
      float h[DT];
      tmem_row<DT>(trow + 128, h);
#pragma unroll
      for (int c = 0; c < DT; ++c) h[c] = real ? h[c] + __ldg(a.seq_b2 + c) : 0.f;
      // InnerTrans layers
      for (int l = 0; l < a.inner_layers; ++l) {
        const float* const* ib = a.inner_bias[l];
        const float* const* ln = a.inner_ln[l];
        float xn[DT];
        layer_norm_row<DT>(h, ln[0], ln[1], xn);
        store_row_canon(sA, row, DT, xn, DT);
        signal();
        wait_d();
        // q, k, v rows; k and v go to smem for the K-1 group peers (adjacent lanes)
        float qv[DT];
        tmem_row<DT>(trow, qv);
        {
          float kv[DT];
          tmem_row<DT>(trow + DT, kv);
#pragma unroll
          for (int c = 0; c < DT; ++c) sKV[row * (2 * DT + 1) + c] = kv[c] + __ldg(ib[1] + c);
          tmem_row<DT>(trow + 2 * DT, kv);
#pragma unroll
          for (int c = 0; c < DT; ++c) sKV[row * (2 * DT + 1) + DT + c] = kv[c] + __ldg(ib[2] + c);
        }
#pragma unroll
        for (int c = 0; c < DT; ++c) qv[c] += __ldg(ib[0] + c);
        __syncwarp();
        const int g0 = row - row % KG;
        float s[KG];
        float mx = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) {
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < DT; ++c) acc = fmaf(qv[c], sKV[(g0 + jj) * (2 * DT + 1) + c], acc);
          s[jj] = acc * scale_in;
          mx = fmaxf(mx, s[jj]);
        }
        float tot = 0.f;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) { s[jj] = __expf(s[jj] - mx); tot += s[jj]; }
        const float inv = 1.f / tot;
        float ctx[DT];
#pragma unroll
        for (int c = 0; c < DT; ++c) {
          float acc = 0.f;
#pragma unroll
          for (int jj = 0; jj < KG; ++jj) acc = fmaf(s[jj], sKV[(g0 + jj) * (2 * DT + 1) + DT + c], acc);
          ctx[c] = acc * inv;
        }
        __syncwarp();
        store_row_canon(sA, row, DT, ctx, DT);
        signal();
        wait_d();
        float o[DT];
        tmem_row<DT>(trow, o);
#pragma unroll
        for (int c = 0; c < DT; ++c) h[c] += o[c] + __ldg(ib[3] + c);       // x1
        layer_norm_row<DT>(h, ln[2], ln[3], xn);
        store_row_canon(sA, row, DT, xn, DT);
        signal();
        wait_d();
#pragma unroll 1
        for (int c0 = 0; c0 < 4 * DT; c0 += 32) {
          float hv[32];
          tmem_row<32>(trow + c0, hv);
#pragma unroll
          for (int u = 0; u < 32; ++u) hv[u] = gelu_f(hv[u] + __ldg(ib[4] + c0 + u));
          store_row_canon(sH, row, 4 * DT, hv, 32, c0);
        }
        signal();
        wait_d();
        tmem_row<DT>(trow + 128, o);
#pragma unroll
        for (int c = 0; c < DT; ++c) h[c] += o[c] + __ldg(ib[5] + c);       // x2
      }
      if (a.inner_layers > 0 && !keep) {
#pragma unroll
        for (int c = 0; c < DT; ++c) h[c] = 0.f;
      }
      if (in_range) {
        float4* dst = reinterpret_cast<float4*>(a.merged + t * DT);
#pragma unroll
        for (int c = 0; c < DT; c += 4) dst[c / 4] = make_float4(h[c], h[c + 1], h[c + 2], h[c + 3]);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

int frontend_supported(int d, int K, int D, int F, int inner_layers) {
  if (!(d == 16 || d == 32)) return 0;
  if (!(K == 2 || K == 4 || K == 8)) return 0;
  if ((2 * D) % 128) return 0;
  if (F > kFP) return 0;
  if (inner_layers > 8) return 0;
  return 1;
}

int frontend_blob_bytes(int d, int D, int F, int inner_layers) {
  (void)F;
  return blob_offsets(d, D, inner_layers).total * 2;
}

void pack_frontend_weights(const float* params, long long tok_w, long long seq_w1, long long seq_w2,
                           const long long (*inner_w)[4], int d, int D, int F, int IL, bf16* blob,
                           cudaStream_t st) {
  const BlobOff o = blob_offsets(d, D, IL);
  PackW pw;
  pw.n = 0;
  auto add = [&](long long src, int in, int out, int n_off, int Kdim, int dst) {
    pw.s[pw.n].src = src; pw.s[pw.n].in = in; pw.s[pw.n].out = out; pw.s[pw.n].n_off = n_off;
    pw.s[pw.n].Kdim = Kdim; pw.s[pw.n].dst = dst; ++pw.n;
  };
  add(tok_w, F, d, 0, kFP, o.tp);
  add(seq_w1, d, 2 * D, 0, d, o.w1);
  add(seq_w2, 2 * D, d, 0, 2 * D, o.w2);
  for (int l = 0; l < IL; ++l) {
    // inner_w[l] = {w_q, w_k, w_v, w_o}; w1/w2 follow b_o in the reference order
    add(inner_w[l][0], d, d, 0, d, o.qkv[l]);
    add(inner_w[l][1], d, d, d, d, o.qkv[l]);
    add(inner_w[l][2], d, d, 2 * d, d, o.qkv[l]);
    add(inner_w[l][3], d, d, 0, d, o.wo[l]);
    add(inner_w[l][3] + (long long)d * d + d, d, 4 * d, 0, d, o.w1i[l]);                       // w1 after b_o
    add(inner_w[l][3] + (long long)d * d + d + 4LL * d * d + 4 * d, 4 * d, d, 0, 4 * d, o.w2i[l]);  // w2 after b1
  }
  pack_canon_kernel<<<dim3(16, pw.n), 256, 0, st>>>(params, pw, blob);
}

template <int DT, int KG>
static int launch_fwd(const FrontArgs& a, cudaStream_t st) {
  const int D = DT * KG;
  const BlobOff bo = blob_offsets(DT, D, a.inner_layers);
  const int smem = ((bo.total + 63) & ~63) * 2 + kTile * kFP * 2 + kTile * 136 * 2 + 64;
  static int done = 0;
  if (!done) {
    cudaFuncSetAttribute(fe_fwd_kernel<DT, KG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 113 * 1024 ? 227 * 1024 : 113 * 1024);
    done = 1;
  }
  const long long ntiles = (a.T + kTile - 1) / kTile;
  const int grid = (int)std::min<long long>(ntiles, 2 * 148);
  fe_fwd_kernel<DT, KG><<<grid, kThreads, smem, st>>>(a);
  return (int)cudaGetLastError();
}

int frontend_fwd(const FrontArgs& a, cudaStream_t st) {
  const int d = a.d, K = a.K;
  if (d == 32 && K == 4) return launch_fwd<32, 4>(a, st);
  if (d == 16 && K == 4) return launch_fwd<16, 4>(a, st);
  if (d == 32 && K == 8) return launch_fwd<32, 8>(a, st);
  if (d == 16 && K == 8) return launch_fwd<16, 8>(a, st);
  if (d == 32 && K == 2) return launch_fwd<32, 2>(a, st);
  if (d == 16 && K == 2) return launch_fwd<16, 2>(a, st);
  return (int)cudaErrorInvalidValue;
}

}  // namespace longer
