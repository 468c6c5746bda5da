// frontend_inner.cu — fused InnerTrans backward (one layer) for 128-token tiles.
//
// Backward of merge_inner_trans (pkg/src/longrec/merge.py:83-112): pre-LN block at width d with
// full attention inside each K-group (grouped_attention, pkg/src/longrec/tensors.py:406-444),
// layer_norm / linear / gelu backward closures (tensors.py:292-404).  The layer is recomputed from
// its saved input h, every contraction is a tcgen05 MMA against smem-resident weights, the four
// weight gradients accumulate in TMEM for the whole kernel (bias gradients ride along as a column
// of ones appended to the contracted activation), and LN / bias column sums use warp transposes.
#include "fe_common.cuh"
#include "frontend.cuh"

#include <algorithm>
#include <cstdlib>

namespace longer {

using namespace fe;

namespace {

// 16-byte vector helpers over bf16 scratch rows (8 values per shared-memory access)
template <int N>
__device__ __forceinline__ void store8_bf16(bf16* dst, const float* v) {
#pragma unroll
  for (int c = 0; c < N; c += 8)
    *reinterpret_cast<uint4*>(dst + c) =
        make_uint4(sm100::pack_bf16(v[c], v[c + 1]), sm100::pack_bf16(v[c + 2], v[c + 3]),
                   sm100::pack_bf16(v[c + 4], v[c + 5]), sm100::pack_bf16(v[c + 6], v[c + 7]));
}
// x (N fp32 values) as packed bf16 pairs
template <int N>
__device__ __forceinline__ void pack_pairs(const float* x, uint32_t* xp) {
#pragma unroll
  for (int c = 0; c < N; c += 2) xp[c / 2] = sm100::pack_bf16(x[c], x[c + 1]);
}
// Σ_c x[c]·row[c] in c order, x as packed bf16 pairs: fp32 += bf16·bf16, one FHFMA per product
template <int N>
__device__ __forceinline__ float dot8_bf16(const uint32_t* xp, const bf16* row) {
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < N; c += 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(row + c);
    acc = sm100::dot2_bf16(xp[c / 2], u.x, acc);
    acc = sm100::dot2_bf16(xp[c / 2 + 1], u.y, acc);
    acc = sm100::dot2_bf16(xp[c / 2 + 2], u.z, acc);
    acc = sm100::dot2_bf16(xp[c / 2 + 3], u.w, acc);
  }
  return acc;
}
// y[c] += a·row[c] with a rounded to bf16 (sm100::bf16_scalar)
template <int N>
__device__ __forceinline__ void axpy8_bf16(float* y, uint32_t a, const bf16* row) {
#pragma unroll
  for (int c = 0; c < N; c += 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(row + c);
    sm100::axpy2_bf16(a, u.x, y[c], y[c + 1]);
    sm100::axpy2_bf16(a, u.y, y[c + 2], y[c + 3]);
    sm100::axpy2_bf16(a, u.z, y[c + 4], y[c + 5]);
    sm100::axpy2_bf16(a, u.w, y[c + 6], y[c + 7]);
  }
}

// NG worker groups: NG = 2 puts two warps on each TMEM lane quadrant (8 workers), each owning half
// of the row's columns (HD = DT / NG); row statistics (LN moments, attention scores, the dP dot
// products, LN-backward sums) meet through a small shared-memory exchange between the pair.
template <int DT, int KG, int NG>
__global__ void __launch_bounds__(32 * (1 + kWorkers * NG), 1) fe_inner_bwd_kernel(FrontArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int XK = DT + 16;                 // activation rows carrying a ones column
  constexpr int F4 = 4 * DT;
  // row length of the FFN tiles sGF / sDF: their weight-gradient MMAs read them MN-major with the
  // hidden units as the M = 128 dimension, so d = 16 (F4 = 64) pads the rows to 128 (the padding
  // columns only feed accumulator rows ≥ F4, which are never read)
  constexpr int FP4 = F4 < 128 ? 128 : F4;
  constexpr int QS = 3 * DT + 8;              // bf16 q|k|v scratch row (16-byte rows; rows 4 apart
                                              // fall in different bank groups)
  constexpr int DCS = DT + 4;                 // fp32 dctx scratch row
  constexpr int HD = DT / NG;                 // columns per worker warp
  constexpr int FH = F4 / NG;                 // FFN hidden columns per worker warp
  const BlobOff bo = blob_offsets(DT, DT * KG, a.inner_layers);
  // weights: forward images [qkv | wo | w1i] and backward images [qkv_n | wo_n | w1i_n | w2i_n]
  bf16* sWf = reinterpret_cast<bf16*>(smem_raw);
  const int nWf = 3 * DT * XK + DT * DT + 4 * DT * XK;   // [Wqkvᵀ|b], Woᵀ, [W1ᵀ|b1]
  const int nWb = 3 * DT * DT + DT * DT + 4 * DT * DT + 4 * DT * DT;
  bf16* sWb = sWf + nWf;
  bf16* w_qkv = sWf;
  bf16* w_wo = w_qkv + 3 * DT * XK;
  bf16* w_w1i = w_wo + DT * DT;
  bf16* w_qkv_n = sWb;
  bf16* w_wo_n = w_qkv_n + 3 * DT * DT;
  bf16* w_w1i_n = w_wo_n + DT * DT;
  bf16* w_w2i_n = w_w1i_n + 4 * DT * DT;
  bf16* sXN = sWb + nWb;                      // 128 x XK
  bf16* sCTX = sXN + kTile * XK;              // 128 x XK
  bf16* sX1N = sCTX + kTile * XK;             // 128 x XK
  bf16* sDX2 = sX1N + kTile * XK;             // 128 x DT
  bf16* sDX1 = sDX2 + kTile * DT;             // 128 x DT
  bf16* sGF = sDX1 + kTile * DT;              // 128 x FP4  (later: dqkv 128 x 3DT)
  bf16* sDF = sGF + kTile * FP4;              // 128 x FP4  (later: dctx fp32 scratch)
  bf16* sDQKV = sGF;
  float* sDC = reinterpret_cast<float*>(sDF); // 128 x DCS
  bf16* sQKV = sDF + kTile * FP4;              // 128 x QS bf16 (q, k, v for the group peers)
  float* sP = reinterpret_cast<float*>(sQKV + kTile * QS);   // NG x 128 x KG (one copy per group)
  float* sS = sP + NG * kTile * KG;                             // NG x 128 x KG (dS)
  float* s_par = sS + NG * kTile * KG;        // [ln1_g, ln1_b, b_o, ln2_g, ln2_b] x DT
  float* sX = s_par + 5 * DT;                 // NG = 2: [2 parity][2 group][128][8] exchange slots
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + (NG > 1 ? 2 * NG * kTile * 8 : 0));
  uint64_t* bar_w = bars;
  uint64_t* bar_a = bars + 1;
  uint64_t* bar_d = bars + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_w, 1);
    sm100::mbar_init(bar_a, 32 * kWorkers * NG);
    sm100::mbar_init(bar_d, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i < 5 * DT; i += blockDim.x) {
    const int v = i / DT, c = i % DT;
    const float* src = v == 0 ? a.inner_ln[0][0] : v == 1 ? a.inner_ln[0][1] : v == 2 ? a.inner_bias[0][3]
                     : v == 3 ? a.inner_ln[0][2] : a.inner_ln[0][3];
    s_par[i] = src[c];
  }
  __syncthreads();
  const uint32_t T_DW2 = tmem;                // F4 rows x DT
  const uint32_t T_DW1 = tmem + 32;           // F4 rows x XK   ([dW1ᵀ | db1])
  const uint32_t T_DWO = tmem + 80;           // DT rows x XK   ([dWoᵀ | dbo])
  const uint32_t T_DWQ = tmem + 128;          // 3DT rows x XK  ([dWqkvᵀ | dbqkv])
  const uint32_t T_W0 = tmem + 176;           // 128: qkv, then f1
  const uint32_t T_W1 = tmem + 304;           // 128: dgf
  const uint32_t T_W2 = tmem + 432;           // 32:  o, dx1n, dctx, dxn
  const long long ntiles = (a.T + kTile - 1) / kTile;

  if (warp == 0) {
    if (lane == 0) {
      sm100::mbar_arrive_expect_tx(bar_w, (nWf + nWb) * 2);
      {
        const uint8_t* src_f = reinterpret_cast<const uint8_t*>(a.wblob + bo.qkv[0]);
        const uint8_t* src_b = reinterpret_cast<const uint8_t*>(a.wblob + bo.qkv_n[0]);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(sm100::smem_u32(sWf)), "l"(src_f), "r"(nWf * 2), "r"(sm100::smem_u32(bar_w)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(sm100::smem_u32(sWb)), "l"(src_b), "r"(nWb * 2), "r"(sm100::smem_u32(bar_w)) : "memory");
      }
      sm100::mbar_wait(bar_w, 0);
      auto S = [](const void* p) { return sm100::smem_u32(p); };
      uint32_t pa = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      bool first = true;
      for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        wait_a();                                                           // xn, dX2
        mma(T_W0, Opnd{S(sXN), XK, 0}, Opnd{S(w_qkv), XK, 0}, XK / 16, 3 * DT, false);
        sm100::mma_commit(bar_d);
        wait_a();                                                           // ctx
        mma(T_W2, Opnd{S(sCTX), XK, 0}, Opnd{S(w_wo), DT, 0}, DT / 16, DT, false);
        sm100::mma_commit(bar_d);
        wait_a();                                                           // x1n
        mma(T_W0, Opnd{S(sX1N), XK, 0}, Opnd{S(w_w1i), XK, 0}, XK / 16, F4, false);
        mma(T_W1, Opnd{S(sDX2), DT, 0}, Opnd{S(w_w2i_n), DT, 0}, DT / 16, F4, false);
        sm100::mma_commit(bar_d);
        // The workers wait only for the dX product of each stage; the weight-gradient MMAs queue
        // behind that commit and are covered by the next one, which precedes any rewrite of
        // their operands (sGF / sDF are reused as dqkv / dctx scratch only after the dx1 commit).
        wait_a();                                                           // gf, df
        mma(T_W2, Opnd{S(sDF), FP4, 0}, Opnd{S(w_w1i_n), F4, 0}, F4 / 16, DT, false);
        sm100::mma_commit(bar_d);
        mma(T_DW2, Opnd{S(sGF), FP4, 1}, Opnd{S(sDX2), DT, 1}, kTile / 16, DT, !first);
        mma(T_DW1, Opnd{S(sDF), FP4, 1}, Opnd{S(sX1N), XK, 1}, kTile / 16, XK, !first);
        wait_a();                                                           // dx1
        mma(T_W2, Opnd{S(sDX1), DT, 0}, Opnd{S(w_wo_n), DT, 0}, DT / 16, DT, false);
        sm100::mma_commit(bar_d);
        mma(T_DWO, Opnd{S(sDX1), DT, 1}, Opnd{S(sCTX), XK, 1}, kTile / 16, XK, !first);
        wait_a();                                                           // dqkv
        mma(T_W2, Opnd{S(sDQKV), 3 * DT, 0}, Opnd{S(w_qkv_n), 3 * DT, 0}, 3 * DT / 16, DT, false);
        mma(T_DWQ, Opnd{S(sDQKV), 3 * DT, 1}, Opnd{S(sXN), XK, 1}, kTile / 16, XK, !first);
        sm100::mma_commit(bar_d);
        first = false;
      }
    }
  } else {
    const int q = warp & 3;
    const int grp = (warp - 1) >> 2;           // column half (NG = 2) of this warp
    const int c0 = grp * HD;
    const int row = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float scale = rsqrtf((float)DT);
    const float* lg1 = s_par;                   // layer vectors staged in shared memory
    const float* lb1 = s_par + DT;
    const float* bo_ = s_par + 2 * DT;
    const float* lg2 = s_par + 3 * DT;
    const float* lb2 = s_par + 4 * DT;
    float* sPg = sP + grp * kTile * KG;         // this group's copy of P and dS
    float* sSg = sS + grp * kTile * KG;
    uint32_t pd = 0;
    auto signal = [&]() { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar_a); };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    // v[0..n) += the pair's partials (a + b == b + a: both warps get bit-identical sums).  Slots
    // alternate by parity, so one barrier per exchange also protects the slot's reuse.
    int xpar = 0;
    auto xsum = [&](float* v, int n) {
      if constexpr (NG > 1) {
        float* mine = sX + ((xpar * NG + grp) * kTile + row) * 8;
        const float* other = sX + ((xpar * NG + (grp ^ 1)) * kTile + row) * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < n) mine[i] = v[i];
        asm volatile("bar.sync %0, 64;" :: "r"(1 + q) : "memory");
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < n) v[i] += other[i];
        xpar ^= 1;
      }
    };
    // LN moments of the row (two-pass, as the reference): mean, then the centred variance
    auto ln_stats = [&](const float* x, float& mu, float& inv) {
      float sm = 0.f;
#pragma unroll
      for (int c = 0; c < HD; ++c) sm += x[c];
      xsum(&sm, 1);
      mu = sm * (1.f / DT);
      float vs = 0.f;
#pragma unroll
      for (int c = 0; c < HD; ++c) { const float t = x[c] - mu; vs += t * t; }
      xsum(&vs, 1);
      inv = rsqrtf(vs * (1.f / DT) + kLnEps);
    };
    auto ones_col = [&](bf16* tile) {           // [· | 1 | 0…] bias column of an XK-wide operand
      if (grp == NG - 1) {
        float pad[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) pad[c] = c == 0 ? 1.f : 0.f;
        store_row(tile, row, XK, pad, 16, DT);
      }
    };
    float cs_l1g = 0.f, cs_l1b = 0.f, cs_l2g = 0.f, cs_l2b = 0.f, cs_b2 = 0.f;   // lane c ↔ column c0 + c
    int my_tiles = 0;
    // R0's rows of tile tl (the warp's 32 rows, its HD columns, of h and dmerged) copied
    // asynchronously into the warp's staging area in the sGF tile — HD / 4 lanes per row, so each
    // instruction covers whole row segments; issued a stage ahead (once sGF is free), no registers
    constexpr int CH = HD / 4, RPI = 32 / CH;          // 16-byte chunks per row, rows per instruction
    float4* const stg = reinterpret_cast<float4*>(sGF) + (warp - 1) * 2 * 32 * CH;
    auto issue_rows = [&](long long tl) {
      const long long tw = tl * kTile + q * 32;         // the warp's first token
#pragma unroll
      for (int k = 0; k < 32 / RPI; ++k) {
        const int r = k * RPI + lane / CH, sg = lane % CH;
        float4* d0 = stg + r * CH + (sg ^ (r & (CH - 1)));
        float4* d1 = d0 + 32 * CH;
        if (tw + r < a.T) {
          sm100::cp_async16(d0, a.h_in + (tw + r) * DT + c0 + 4 * sg);
          sm100::cp_async16(d1, a.dmerged + (tw + r) * DT + c0 + 4 * sg);
        } else {
          *d0 = make_float4(0.f, 0.f, 0.f, 0.f);
          *d1 = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      sm100::cp_async_commit();
    };
    if (blockIdx.x < ntiles) issue_rows(blockIdx.x);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++my_tiles) {
      const long long t = tile * kTile + row;
      const bool in_range = t < a.T;
      bool keep = false;
      if (in_range) {
        const int b = (int)(t / a.Lp), j = (int)(t % a.Lp);
        const int n = min(max(a.n_events[b], 0), a.L);
        keep = (j / a.K) >= (a.Lp - n) / a.K;
      }
      // ---- R0: x = h; LN1; dX2 = dmerged ⊙ keep
      // The warp's 32 rows (its HD columns) of h and dmerged are loaded cooperatively — HD / 4
      // lanes per row, so each instruction covers whole row segments — into a staging area in the
      // (free: R5's MMAs are done) sGF tile, then each thread takes its own row.
      float h[HD], dx2[HD];
      {
        sm100::cp_async_wait_all();                       // this tile's rows (issued a stage ahead)
        __syncwarp();
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const float4 hv = stg[lane * CH + (j ^ (lane & (CH - 1)))];
          const float4 dv = keep ? stg[32 * CH + lane * CH + (j ^ (lane & (CH - 1)))] : make_float4(0.f, 0.f, 0.f, 0.f);
          h[4 * j] = hv.x; h[4 * j + 1] = hv.y; h[4 * j + 2] = hv.z; h[4 * j + 3] = hv.w;
          dx2[4 * j] = dv.x; dx2[4 * j + 1] = dv.y; dx2[4 * j + 2] = dv.z; dx2[4 * j + 3] = dv.w;
        }
        __syncwarp();
      }
      float mu1, inv1;
      ln_stats(h, mu1, inv1);
      {
        float xn[HD];
#pragma unroll
        for (int c = 0; c < HD; ++c) xn[c] = (h[c] - mu1) * inv1 * lg1[c0 + c] + lb1[c0 + c];
        store_row(sXN, row, XK, xn, HD, c0);
      }
      ones_col(sXN);
      store_row(sDX2, row, DT, dx2, HD, c0);
      signal();
      // the next tile's h / dmerged rows into L2 while this one runs (register-free: a register
      // prefetch spills at the 168-register ceiling), so its R0 loads hit L2 instead of HBM
      {
        const long long tn = (tile + gridDim.x) * kTile + row;
        if (grp == 0 && tn < a.T) {
          sm100::prefetch_l2(a.h_in + tn * DT);
          sm100::prefetch_l2(a.dmerged + tn * DT);
        }
      }
      // ---- R1: q, k, v; group attention (scratch keeps q|k|v (bf16) and P (fp32) for the peers)
      wait_d();
      uint32_t qp[HD / 2];                       // q as bf16 pairs (the scores' operand)
      {
        float kvv[HD];
        tmem_row<HD>(T_W0 + lo + c0, kvv);
        pack_pairs<HD>(kvv, qp);
        bf16* qs = sQKV + row * QS;
#pragma unroll
        for (int c = 0; c < HD; c += 8)
          *reinterpret_cast<uint4*>(qs + c0 + c) = make_uint4(qp[c / 2], qp[c / 2 + 1], qp[c / 2 + 2], qp[c / 2 + 3]);
        tmem_row<HD>(T_W0 + lo + DT + c0, kvv);
        store8_bf16<HD>(qs + DT + c0, kvv);
        tmem_row<HD>(T_W0 + lo + 2 * DT + c0, kvv);
        store8_bf16<HD>(qs + 2 * DT + c0, kvv);
      }
      __syncwarp();
      const int g0 = row - row % KG;
      const int me = row - g0;
      float p[KG];
      {
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) p[jj] = dot8_bf16<HD>(qp, sQKV + (g0 + jj) * QS + DT + c0);
        xsum(p, KG);
        float mx = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) { p[jj] *= scale; mx = fmaxf(mx, p[jj]); }
        float tot = 0.f;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) { p[jj] = __expf(p[jj] - mx); tot += p[jj]; }
        const float rinv = 1.f / tot;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) { p[jj] *= rinv; sPg[row * KG + jj] = p[jj]; }
      }
      {
        float ctx[HD];
#pragma unroll
        for (int c = 0; c < HD; ++c) ctx[c] = 0.f;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) axpy8_bf16<HD>(ctx, sm100::bf16_scalar(p[jj]), sQKV + (g0 + jj) * QS + 2 * DT + c0);
        store_row(sCTX, row, XK, ctx, HD, c0);
      }
      ones_col(sCTX);
      signal();
      // ---- R2: x1 = h + ctx·Wo + bo; LN2
      wait_d();
      float x1[HD];
      tmem_row<HD>(T_W2 + lo + c0, x1);
#pragma unroll
      for (int c = 0; c < HD; ++c) x1[c] += h[c] + bo_[c0 + c];
      float mu2, inv2;
      ln_stats(x1, mu2, inv2);
      {
        float x1n[HD];
#pragma unroll
        for (int c = 0; c < HD; ++c) x1n[c] = (x1[c] - mu2) * inv2 * lg2[c0 + c] + lb2[c0 + c];
        store_row(sX1N, row, XK, x1n, HD, c0);
      }
      ones_col(sX1N);
      signal();
      // ---- R3: FFN: gf = GELU(f1), df = (dX2·W2ᵀ) ⊙ GELU'(f1)   (this warp: FH hidden columns)
      wait_d();
#pragma unroll 1
      for (int cc = grp * FH; cc < grp * FH + FH; cc += 32) {
        float fv[32], gv[32];
        tmem_row2<32>(T_W0 + lo + cc, fv, T_W1 + lo + cc, gv);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          float gd;                                                   // b1 added by the MMA
          fv[u] = gelu_and_grad(fv[u], gd);
          gv[u] *= gd;
        }
        store_row(sGF, row, FP4, fv, 32, cc);
        store_row(sDF, row, FP4, gv, 32, cc);
      }
      signal();
      // ---- R4: LN2 backward → dx1 = dX2 + LN2ᵀ(dx1n)
      wait_d();
      float g[HD], xh[HD], dx1[HD], tmp[HD];
      tmem_row<HD>(T_W2 + lo + c0, g);                                // dx1n
      {
        float m[2] = {0.f, 0.f};
#pragma unroll
        for (int c = 0; c < HD; ++c) {
          xh[c] = (x1[c] - mu2) * inv2;
          const float gh = g[c] * lg2[c0 + c];
          m[0] += gh;
          m[1] += gh * xh[c];
        }
        xsum(m, 2);
        const float m1 = m[0] * (1.f / DT), m2 = m[1] * (1.f / DT);
#pragma unroll
        for (int c = 0; c < HD; ++c) {
          dx1[c] = dx2[c] + (g[c] * lg2[c0 + c] - m1 - xh[c] * m2) * inv2;
          tmp[c] = g[c] * xh[c];
        }
      }
      cs_l2g += warp_colsum<HD>(tmp);
      cs_l2b += warp_colsum<HD>(g);
      cs_b2 += warp_colsum<HD>(dx2);
      store_row(sDX1, row, DT, dx1, HD, c0);
      signal();
      // ---- R5: dctx → group attention backward → dqkv
      wait_d();
      {
        float dc[HD];
        tmem_row<HD>(T_W2 + lo + c0, dc);
#pragma unroll
        for (int c = 0; c < HD; c += 4)
          *reinterpret_cast<float4*>(sDC + row * DCS + c0 + c) = make_float4(dc[c], dc[c + 1], dc[c + 2], dc[c + 3]);
        float dp[KG];
        uint32_t dcp[HD / 2];
        pack_pairs<HD>(dc, dcp);
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) dp[jj] = dot8_bf16<HD>(dcp, sQKV + (g0 + jj) * QS + 2 * DT + c0);
        xsum(dp, KG);
        float D = 0.f;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) D += dp[jj] * p[jj];
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) sSg[row * KG + jj] = p[jj] * (dp[jj] - D) * scale;
      }
      __syncwarp();
      {
        float dqkv[3 * HD];
#pragma unroll
        for (int c = 0; c < 3 * HD; ++c) dqkv[c] = 0.f;
#pragma unroll
        for (int jj = 0; jj < KG; ++jj) {         // same per-element summation order as a c-outer loop
          const bf16* pr = sQKV + (g0 + jj) * QS;
          axpy8_bf16<HD>(dqkv, sm100::bf16_scalar(sSg[row * KG + jj]), pr + DT + c0);           // dq += dS_ij k_j
          axpy8_bf16<HD>(dqkv + HD, sm100::bf16_scalar(sSg[(g0 + jj) * KG + me]), pr + c0);     // dk += dS_ji q_j
          const float pj = sPg[(g0 + jj) * KG + me];                        // dv += P_ji dctx_j
          const float* dcr = sDC + (g0 + jj) * DCS + c0;
#pragma unroll
          for (int c = 0; c < HD; c += 4) {
            const float4 d4 = *reinterpret_cast<const float4*>(dcr + c);
            dqkv[2 * HD + c] = fmaf(pj, d4.x, dqkv[2 * HD + c]);
            dqkv[2 * HD + c + 1] = fmaf(pj, d4.y, dqkv[2 * HD + c + 1]);
            dqkv[2 * HD + c + 2] = fmaf(pj, d4.z, dqkv[2 * HD + c + 2]);
            dqkv[2 * HD + c + 3] = fmaf(pj, d4.w, dqkv[2 * HD + c + 3]);
          }
        }
        __syncwarp();
        store_row(sDQKV, row, 3 * DT, dqkv, HD, c0);
        store_row(sDQKV, row, 3 * DT, dqkv + HD, HD, DT + c0);
        store_row(sDQKV, row, 3 * DT, dqkv + 2 * HD, HD, 2 * DT + c0);
      }
      signal();
      // ---- R6: LN1 backward → dh = dx1 + LN1ᵀ(dxn)
      wait_d();
      // the dqkv MMAs (the last readers of sGF) are done: the next tile's R0 rows start arriving
      if (tile + gridDim.x < ntiles) issue_rows(tile + gridDim.x);
      tmem_row<HD>(T_W2 + lo + c0, g);                                // dxn
      {
        float m[2] = {0.f, 0.f};
#pragma unroll
        for (int c = 0; c < HD; ++c) {
          xh[c] = (h[c] - mu1) * inv1;
          const float gh = g[c] * lg1[c0 + c];
          m[0] += gh;
          m[1] += gh * xh[c];
        }
        xsum(m, 2);
        const float m1 = m[0] * (1.f / DT), m2 = m[1] * (1.f / DT);
#pragma unroll
        for (int c = 0; c < HD; ++c) {
          dx1[c] += (g[c] * lg1[c0 + c] - m1 - xh[c] * m2) * inv1;
          tmp[c] = g[c] * xh[c];
        }
      }
      cs_l1g += warp_colsum<HD>(tmp);
      cs_l1b += warp_colsum<HD>(g);
      if (in_range) {
        if (a.dh_out_bf) {
          store8_bf16<HD>(a.dh_out_bf + t * DT + c0, dx1);
        } else {
#pragma unroll
          for (int c = 0; c < HD; c += 4)
            *reinterpret_cast<float4*>(a.dh_out + t * DT + c0 + c) = make_float4(dx1[c], dx1[c + 1], dx1[c + 2], dx1[c + 3]);
        }
      }
    }
    // ---- flush this CTA's accumulators (gradient slots: 0 w_q,1 b_q,2 w_k,3 b_k,4 w_v,5 b_v,
    //      6 w_o,7 b_o,8 w1,9 b1,10 w2,11 b2,12 ln1_g,13 ln1_b,14 ln2_g,15 ln2_b); each warp
    //      flushes its column half, the last group the bias column
    if (my_tiles > 0) {
      float* const* G = a.g_inner;
      const bool bias_col = grp == NG - 1;
      float w[HD], wb[16];
      {   // dW2 [4d][d]: TMEM row f = hidden unit
        tmem_row<HD>(T_DW2 + lo + c0, w);
        if (row < F4) {
#pragma unroll
          for (int c = 0; c < HD; ++c) atomicAdd(G[10] + row * DT + c0 + c, w[c]);
        }
      }
      {   // [dW1ᵀ | db1]: row f = hidden unit
        tmem_row<HD>(T_DW1 + lo + c0, w);
        tmem_row<16>(T_DW1 + lo + DT, wb);
        if (row < F4) {
#pragma unroll
          for (int c = 0; c < HD; ++c) atomicAdd(G[8] + (c0 + c) * F4 + row, w[c]);
          if (bias_col) atomicAdd(G[9] + row, wb[0]);
        }
      }
      {   // [dWoᵀ | dbo]: row c = output column of W_o (first DT rows valid)
        tmem_row<HD>(T_DWO + lo + c0, w);
        tmem_row<16>(T_DWO + lo + DT, wb);
        if (row < DT) {
#pragma unroll
          for (int k = 0; k < HD; ++k) atomicAdd(G[6] + (c0 + k) * DT + row, w[k]);
          if (bias_col) atomicAdd(G[7] + row, wb[0]);
        }
      }
      {   // [dWqkvᵀ | dbqkv]: row o ∈ [0, 3d)
        tmem_row<HD>(T_DWQ + lo + c0, w);
        tmem_row<16>(T_DWQ + lo + DT, wb);
        if (row < 3 * DT) {
          const int which = row / DT, oc = row % DT;
#pragma unroll
          for (int k = 0; k < HD; ++k) atomicAdd(G[2 * which] + (c0 + k) * DT + oc, w[k]);
          if (bias_col) atomicAdd(G[2 * which + 1] + oc, wb[0]);
        }
      }
      if (lane < HD) {
        atomicAdd(G[12] + c0 + lane, cs_l1g);
        atomicAdd(G[13] + c0 + lane, cs_l1b);
        atomicAdd(G[14] + c0 + lane, cs_l2g);
        atomicAdd(G[15] + c0 + lane, cs_l2b);
        atomicAdd(G[11] + c0 + lane, cs_b2);
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

template <int DT, int KG, int NG>
int launch_inner_bwd_ng(const FrontArgs& a, cudaStream_t st) {
  constexpr int XK = DT + 16, F4 = 4 * DT, FP4 = F4 < 128 ? 128 : F4, QS = 3 * DT + 8;
  const int nW = 7 * DT * XK + DT * DT + 12 * DT * DT;
  const int smem = nW * 2 + kTile * (3 * XK + 2 * DT + 2 * FP4 + QS) * 2 + NG * kTile * KG * 8 + 5 * DT * 4 +
                   (NG > 1 ? 2 * NG * kTile * 8 * 4 : 0) + 64;
  if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;
  smem_attr(fe_inner_bwd_kernel<DT, KG, NG>, 227 * 1024);
  const long long ntiles = (a.T + kTile - 1) / kTile;
  int grid = (int)std::min<long long>(ntiles, 148);
  if (g_knobs.fe_grid > 0) grid = std::min(grid, g_knobs.fe_grid);   // testing: many tiles per CTA
  g_launch_fence = kFenceFrontIn | kFenceFrontOut;
  launch(fe_inner_bwd_kernel<DT, KG, NG>, grid, 32 * (1 + kWorkers * NG), std::max(smem, 116 * 1024), st, a);
  return (int)cudaGetLastError();
}

// head width 32: eight workers (column pairs); 16: four
template <int DT, int KG>
int launch_inner_bwd(const FrontArgs& a, cudaStream_t st) {
  return launch_inner_bwd_ng<DT, KG, DT == 32 ? 2 : 1>(a, st);
}

}  // namespace

int frontend_inner_bwd(const FrontArgs& a, cudaStream_t st) {
  if (a.inner_layers != 1) return (int)cudaErrorInvalidValue;
  if (a.d == 32 && a.K == 4) return launch_inner_bwd<32, 4>(a, st);
  if (a.d == 16 && a.K == 4) return launch_inner_bwd<16, 4>(a, st);
  if (a.d == 32 && a.K == 8) return launch_inner_bwd<32, 8>(a, st);
  if (a.d == 16 && a.K == 8) return launch_inner_bwd<16, 8>(a, st);
  if (a.d == 32 && a.K == 2) return launch_inner_bwd<32, 2>(a, st);
  if (a.d == 16 && a.K == 2) return launch_inner_bwd<16, 2>(a, st);
  return (int)cudaErrorInvalidValue;
}

}  // namespace longer
