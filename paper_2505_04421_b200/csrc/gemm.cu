// gemm.cu — generic tcgen05 GEMM with fused epilogues. See gemm.cuh for the contract.
//
// CTA = 1 TMA warp + 1 MMA warp (also owns TMEM) + 8 epilogue warps, persistent over work items
// with a double-buffered TMEM accumulator.  The smem ring depth is a template parameter chosen from
// the K extent (1, 2 or 4 stages); the epilogue stores go through a per-warp smem transpose.
#include "gemm.cuh"
#include "sm100.cuh"
#include "tma.cuh"
#include "common.cuh"

#include <algorithm>
#include <cstdlib>

namespace longer {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN, int STAGES>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STG_BYTES = 4096;             // per epilogue warp: a 32 x 32 fp32 chunk
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + 8 * STG_BYTES;
};

// Persistent: a CTA walks work items w = blockIdx.x + i·gridDim.x over (n-tile, m-tile, k-split).
// The TMA ring runs continuously across items and the accumulator is double-buffered in TMEM
// (2·BN columns), so the MMAs and loads of item i+1 overlap the epilogue of item i.
//   tmem_full[b]  MMA → epilogue: buffer b holds a finished item (b = local item index & 1)
//   tmem_empty[b] epilogue → MMA: buffer b drained (8 arrivals, one per epilogue warp)
// Each buffer's barriers alternate strictly, so no phase can be skipped.
template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            GemmArgs g, int kb_per_split, int n_tiles, int m_tiles, int n_items) {
  using S = Smem<BN, STAGES>;
  constexpr uint32_t TCOLS = 2 * BN < 32 ? 32 : 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;            // [2]
  uint64_t* tmem_empty = tmem_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32;
  const int nkb_total = (g.K + BK - 1) / BK;
  auto item = [&](int w, int& n0, int& m0, int& kb_begin, int& nkb) {
    const int x = w % n_tiles, y = (w / n_tiles) % m_tiles, z = w / (n_tiles * m_tiles);
    n0 = x * BN;
    m0 = y * BM;
    kb_begin = z * kb_per_split;
    nkb = min(nkb_total, kb_begin + kb_per_split) - kb_begin;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { sm100::mbar_init(&tmem_full[b], 1); sm100::mbar_init(&tmem_empty[b], kEpiWarps); }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<TCOLS>(tmem_slot);
  if (warp == 0 && threadIdx.x == 0) {             // descriptors are kernel parameters: before the wait
    sm100::tma_prefetch(&tmA);
    sm100::tma_prefetch(&tmB);
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // LONGER_GEMM_LATE_TRIGGER: dependents launch once this CTA has issued its last MMA (instead of
  // at its start), so their CTAs do not sit on the SMs through the whole GEMM
  if (!g.late_trigger) pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (sm100::elect_one()) {
      int it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        int n0, m0, kb_begin, nkb;
        item(w, n0, m0, kb_begin, nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % STAGES, round = it / STAGES;
          if (it >= STAGES) sm100::mbar_wait(&empty[s], (round - 1) & 1);
          uint8_t* sa = smem + s * S::STAGE_BYTES;
          uint8_t* sb = sa + S::A_BYTES;
          sm100::mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
          const int k0 = (kb_begin + i) * BK;
          if (!g.a_mn_major) {
            sm100::tma_load_2d(sa, &tmA, &full[s], k0, m0);
          } else {
            sm100::tma_load_2d(sa, &tmA, &full[s], m0, k0);
            sm100::tma_load_2d(sa + 8192, &tmA, &full[s], m0 + 64, k0);
          }
          if (!g.b_mn_major) {
            sm100::tma_load_2d(sb, &tmB, &full[s], k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) sm100::tma_load_2d(sb + j * 8192, &tmB, &full[s], n0 + 64 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (sm100::elect_one()) {
      const uint32_t idesc = sm100::make_idesc_bf16(BM, BN, g.a_mn_major, g.b_mn_major);
      int it = 0, j = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++j) {
        int n0, m0, kb_begin, nkb;
        item(w, n0, m0, kb_begin, nkb);
        const int buf = j & 1;
        if (j >= 2) {                                 // the epilogue has drained this buffer
          sm100::mbar_wait(&tmem_empty[buf], ((j >> 1) - 1) & 1);
          sm100::tc_fence_after();
        }
        const uint32_t acc = tmem + (uint32_t)(buf * BN);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % STAGES, round = it / STAGES;
          sm100::mbar_wait(&full[s], round & 1);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(smem + s * S::STAGE_BYTES);
          const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            uint64_t ad = g.a_mn_major ? sm100::make_sdesc(sa + kk * 2048, 8192, 1024, sm100::LAYOUT_SW128)
                                       : sm100::make_sdesc(sa + kk * 32, 16, 1024, sm100::LAYOUT_SW128);
            uint64_t bd = g.b_mn_major ? sm100::make_sdesc(sb + kk * 2048, 8192, 1024, sm100::LAYOUT_SW128)
                                       : sm100::make_sdesc(sb + kk * 32, 16, 1024, sm100::LAYOUT_SW128);
            sm100::mma_bf16(acc, ad, bd, idesc, (i | kk) != 0);
          }
          sm100::mma_commit(&empty[s]);
        }
        sm100::mma_commit(&tmem_full[buf]);
      }
      if (g.late_trigger) pdl_trigger();
    }
  } else {
    // Epilogue warps e = 0..7: TMEM lane quarter q = warp % 4, column chunks c ≡ e/4 (mod 2).
    // Thread = output row: the 32 accumulators of a chunk are processed in registers and every
    // global access is a 16-byte vector (bf16 x 8 / fp32 x 4); flag tests run once per chunk.
    const int e = warp - 2;
    const int q = warp & 3;
    const int lane = threadIdx.x & 31;
    // Staged stores: the warp's 32 rows x 32 columns go through its own smem buffer (XOR-swizzled
    // 16-byte segments, conflict-free both ways) and leave as whole 64 / 128-byte row segments, so
    // each store instruction fills its sectors instead of writing 16 bytes into 32 different rows.
    uint4* stg = reinterpret_cast<uint4*>(smem + STAGES * S::STAGE_BYTES + 256 + e * S::STG_BYTES);
    const bool staged = g.staged != 0;
    auto store_bf16 = [&](void* base, int ld, int m_base, int nb, const float* v) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        stg[lane * 4 + (j ^ ((lane >> 1) & 3))] =
            make_uint4(sm100::pack_bf16(v[8 * j], v[8 * j + 1]), sm100::pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                       sm100::pack_bf16(v[8 * j + 4], v[8 * j + 5]), sm100::pack_bf16(v[8 * j + 6], v[8 * j + 7]));
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = k * 8 + (lane >> 2), sgm = lane & 3;
        const uint4 val = stg[r * 4 + (sgm ^ ((r >> 1) & 3))];
        if (m_base + r < g.M)
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + (size_t)(m_base + r) * ld + nb + sgm * 8) = val;
      }
      __syncwarp();
    };
    auto store_f32 = [&](float* base, int ld, int m_base, int nb, const float* v) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        stg[lane * 8 + (j ^ (lane & 7))] = make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                                                      __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = k * 4 + (lane >> 3), sgm = lane & 7;
        const uint4 val = stg[r * 8 + (sgm ^ (r & 7))];
        if (m_base + r < g.M) *reinterpret_cast<uint4*>(base + (size_t)(m_base + r) * ld + nb + sgm * 4) = val;
      }
      __syncwarp();
    };
    int j = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++j) {
    int n0, m0, kb_begin_unused, nkb_unused;
    item(w, n0, m0, kb_begin_unused, nkb_unused);
    const int buf = j & 1;
    const uint32_t flags = g.flags;
    // bias of this warp's column chunks, one value per lane (broadcast by shuffles below), loaded
    // before the accumulator wait so the load latency hides behind the MMAs
    constexpr int NCH = (BN + 63) / 64;
    float bias_l[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int col = n0 + (e >> 2) * 32 + 64 * k + lane;
      bias_l[k] = ((flags & EPI_BIAS) && col < g.N) ? __ldg(g.bias + col) : 0.f;
    }
    // one column chunk per warp (BN = 64): the residual row chunk is loaded before the wait too
    float res_pre[NCH == 1 ? 32 : 1];
    const bool res_early = NCH == 1 && (flags & EPI_RESID) && staged;
    if constexpr (NCH == 1) {
      const int col = n0 + (e >> 2) * 32;
      const int rr = m0 + q * 32 + lane;
      if (res_early && col + 32 <= g.N && rr < g.M) {
        const float4* rp = reinterpret_cast<const float4*>(g.resid + (size_t)rr * g.ldr + col);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float4 r4 = rp[t];
          res_pre[4 * t] = r4.x; res_pre[4 * t + 1] = r4.y; res_pre[4 * t + 2] = r4.z; res_pre[4 * t + 3] = r4.w;
        }
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t) res_pre[t] = 0.f;
      }
    }
    sm100::mbar_wait(&tmem_full[buf], (j >> 1) & 1);
    sm100::tc_fence_after();
    const uint32_t tmem_acc = tmem + (uint32_t)(buf * BN);
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < g.M;
    const float rmask = ((flags & EPI_ROWMASK) && row_ok) ? g.rowmask[row] : 1.f;
#pragma unroll 1
    for (int c = (e >> 2) * 32; c < BN; c += 64) {
      uint32_t r[32];
      sm100::tmem_ld32(tmem_acc + ((uint32_t)(q * 32) << 16) + c, r);
      sm100::tmem_ld_wait();
      sm100::reg_fence(r);
      const int nb = n0 + c;
      if (nb >= g.N) continue;                                   // warp-uniform
      const int m_base = m0 + q * 32;
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      if (staged && nb + 32 <= g.N) {
        // warp-collective path: rows past M compute on zeros and are never stored
        if (flags & EPI_BIAS) {
          float bl = bias_l[0];
#pragma unroll
          for (int k = 1; k < NCH; ++k)
            if (c == (e >> 2) * 32 + 64 * k) bl = bias_l[k];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += __shfl_sync(0xffffffffu, bl, j);
        }
        if (flags & EPI_SAVE_PRE) store_bf16(g.pre_bf16, g.ldc_bf, m_base, nb, v);
        if (flags & EPI_GELU) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
        }
        if ((flags & EPI_GELU_BWD) && row_ok) {
          const uint4* pp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(g.pre_bf16) +
                                                           (size_t)row * g.ldc_bf + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 p4 = pp[j];
            const uint32_t w[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              v[8 * j + 2 * u] *= gelu_grad_f(sm100::bf16_lo(w[u]));
              v[8 * j + 2 * u + 1] *= gelu_grad_f(sm100::bf16_hi(w[u]));
            }
          }
        }
        if (res_early) {
          if constexpr (NCH == 1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += res_pre[j];
          }
        } else if ((flags & EPI_RESID) && row_ok) {
          const float4* rp = reinterpret_cast<const float4*>(g.resid + (size_t)row * g.ldr + nb);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 r4 = rp[j];
            v[4 * j] += r4.x; v[4 * j + 1] += r4.y; v[4 * j + 2] += r4.z; v[4 * j + 3] += r4.w;
          }
        }
        if (flags & EPI_ROWMASK) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= rmask;
        }
        if (flags & EPI_OUT_F32) {
          if (flags & EPI_ATOMIC) {
            if (row_ok) {
              float4* cp = reinterpret_cast<float4*>(g.C + (size_t)row * g.ldc + nb);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                atomicAdd(cp + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
            }
          } else {
            store_f32(g.C, g.ldc, m_base, nb, v);
          }
        }
        if (flags & EPI_OUT_BF16) store_bf16(g.C_bf16, g.ldc_bf, m_base, nb, v);
        continue;
      }
      if (!row_ok) continue;
      if (nb + 32 <= g.N) {
        if (flags & EPI_BIAS) {
          const float4* bp = reinterpret_cast<const float4*>(g.bias + nb);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 b4 = __ldg(bp + j);
            v[4 * j] += b4.x; v[4 * j + 1] += b4.y; v[4 * j + 2] += b4.z; v[4 * j + 3] += b4.w;
          }
        }
        if (flags & EPI_SAVE_PRE) {
          uint4* pp = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(g.pre_bf16) + (size_t)row * g.ldc_bf + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            pp[j] = make_uint4(sm100::pack_bf16(v[8 * j], v[8 * j + 1]), sm100::pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                               sm100::pack_bf16(v[8 * j + 4], v[8 * j + 5]), sm100::pack_bf16(v[8 * j + 6], v[8 * j + 7]));
        }
        if (flags & EPI_GELU) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
        }
        if (flags & EPI_GELU_BWD) {
          const uint4* pp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(g.pre_bf16) +
                                                           (size_t)row * g.ldc_bf + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 p4 = pp[j];
            const uint32_t w[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              v[8 * j + 2 * u] *= gelu_grad_f(sm100::bf16_lo(w[u]));
              v[8 * j + 2 * u + 1] *= gelu_grad_f(sm100::bf16_hi(w[u]));
            }
          }
        }
        if (flags & EPI_RESID) {
          const float4* rp = reinterpret_cast<const float4*>(g.resid + (size_t)row * g.ldr + nb);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 r4 = rp[j];
            v[4 * j] += r4.x; v[4 * j + 1] += r4.y; v[4 * j + 2] += r4.z; v[4 * j + 3] += r4.w;
          }
        }
        if (flags & EPI_ROWMASK) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= rmask;
        }
        if (flags & EPI_OUT_F32) {
          float4* cp = reinterpret_cast<float4*>(g.C + (size_t)row * g.ldc + nb);
          if (flags & EPI_ATOMIC) {
#pragma unroll
            for (int j = 0; j < 8; ++j) atomicAdd(cp + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) cp[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
        }
        if (flags & EPI_OUT_BF16) {
          uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(g.C_bf16) + (size_t)row * g.ldc_bf + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            op[j] = make_uint4(sm100::pack_bf16(v[8 * j], v[8 * j + 1]), sm100::pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                               sm100::pack_bf16(v[8 * j + 4], v[8 * j + 5]), sm100::pack_bf16(v[8 * j + 6], v[8 * j + 7]));
        }
      } else {
        // ragged last chunk: scalar path
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = nb + j;
          if (n >= g.N) continue;
          float x = v[j];
          if (flags & EPI_BIAS) x += g.bias[n];
          if (flags & EPI_SAVE_PRE)
            reinterpret_cast<__nv_bfloat16*>(g.pre_bf16)[(size_t)row * g.ldc_bf + n] = __float2bfloat16(x);
          if (flags & EPI_GELU) x = gelu_f(x);
          if (flags & EPI_GELU_BWD)
            x *= gelu_grad_f(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(g.pre_bf16)[(size_t)row * g.ldc_bf + n]));
          if (flags & EPI_RESID) x += g.resid[(size_t)row * g.ldr + n];
          x *= rmask;
          if (flags & EPI_OUT_F32) {
            float* dst = g.C + (size_t)row * g.ldc + n;
            if (flags & EPI_ATOMIC) atomicAdd(dst, x); else *dst = x;
          }
          if (flags & EPI_OUT_BF16)
            reinterpret_cast<__nv_bfloat16*>(g.C_bf16)[(size_t)row * g.ldc_bf + n] = __float2bfloat16(x);
        }
      }
    }
    // this item's accumulator is drained: hand the buffer back to the MMA warp
    sm100::tc_fence_before();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&tmem_empty[buf]);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<(2 * BN < 32 ? 32 : 2 * BN)>(tmem);
}

template <int BN, int STAGES>
int launch_cfg(const GemmArgs& g, const CUtensorMap& tA, const CUtensorMap& tB, dim3 grid, int kb_per,
               cudaStream_t st) {
  const int smem = Smem<BN, STAGES>::TOTAL;
  smem_attr(gemm_kernel<BN, STAGES>, smem);
  const int n_items = (int)(grid.x * grid.y * grid.z);
  const int ctas = std::min(n_items, 148);
  GemmArgs ga = g;
  if (ga.staged < 0) ga.staged = g_knobs.gemm_stage ? 1 : 0;
  ga.late_trigger = g_knobs.gemm_late_trigger;
  g_launch_fence = kFenceGemmIn | kFenceGemmOut;
  launch(gemm_kernel<BN, STAGES>, dim3(ctas), kThreads, smem, st, tA, tB, ga, kb_per, (int)grid.x, (int)grid.y,
         n_items);
  return (int)cudaGetLastError();
}

template <int BN>
int launch_bn(const GemmArgs& g, cudaStream_t st) {
  CUtensorMap tA, tB;
  int rc;
  if (!g.a_mn_major) rc = tma::encode_2d_bf16(&tA, g.A, g.K, g.M, g.lda, BK, BM);
  else rc = tma::encode_2d_bf16(&tA, g.A, g.M, g.K, g.lda, 64, BK);
  if (rc) return rc;
  if (!g.b_mn_major) rc = tma::encode_2d_bf16(&tB, g.B, g.K, g.N, g.ldb, BK, BN);
  else rc = tma::encode_2d_bf16(&tB, g.B, g.N, g.K, g.ldb, 64, BK);
  if (rc) return rc;
  const int nkb = (g.K + BK - 1) / BK;
  const int tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM);
  int want = g.split_k;
  // split-K for the weight gradients: about 37 items (74 in round 1; equal at c2 and 15 us better at
  // c5 at the end of round 2) (the persistent CTAs stream their k-blocks back
  // to back; more splits only multiply the atomic epilogues, and these GEMMs run beside other
  // kernels on the side stream: 296 → 148 → 74 items measured 1.648 → 1.640 → 1.625 ms per step).
  // LONGER_SPLIT_ITEMS overrides the target.
  const int split_items = g_knobs.split_items;
  if (want == 0) want = (g.flags & EPI_ATOMIC) ? std::max(1, std::min(split_items / tiles, nkb / 4)) : 1;
  int split = std::max(1, std::min(want, nkb));
  int kb_per = (nkb + split - 1) / split;
  split = (nkb + kb_per - 1) / kb_per;
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, split);
  if (kb_per <= 1) return launch_cfg<BN, 1>(g, tA, tB, grid, kb_per, st);
  if (kb_per <= 2) return launch_cfg<BN, 2>(g, tA, tB, grid, kb_per, st);
  return launch_cfg<BN, 4>(g, tA, tB, grid, kb_per, st);
}

}  // namespace

int gemm_launch(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return 0;
  if (g.split_k != 1 && !(g.flags & EPI_ATOMIC)) return (int)cudaErrorInvalidValue;
  // Widest tile that still gives the 148 SMs work: the query-row GEMMs (M = 8,960 → 70 row
  // tiles) would otherwise leave half the machine idle at N ≤ 128.  "Enough work" is ≥ 200 tiles:
  // the query-row QKV / FFN-up GEMMs (N = 384 / 512) then take 128-wide tiles (210 / 280 items
  // over 148 CTAs, the TMEM double buffer overlapping epilogues) instead of 140 256-wide ones
  // (step 1.574 → 1.570 ms; 60 / 120 / 300 measured slower).
  const long long mt = (g.M + BM - 1) / BM;
  auto tiles = [&](int bn) { return mt * ((g.N + bn - 1) / bn); };
  const bool split = (g.flags & EPI_ATOMIC) != 0;           // split-K fills the machine itself
  if (g.N <= 64) return launch_bn<64>(g, st);
  // LONGER_GEMM_MIN_TILES overrides both thresholds (read per call; 1 forces the widest tile)
  // (auto: 60 when K and N are both >= 256 — c5's query-row GEMMs, where each narrower tile re-reads
  // a 64 KB A tile: 6.73 -> 6.67 ms; at c2's K = 128 the 200 threshold measured best)
  const int min_tiles = g_knobs.gemm_min_tiles > 0 ? g_knobs.gemm_min_tiles : (g.K >= 256 && g.N >= 256 ? 60 : 200);
  const int min_tiles128 = std::min(min_tiles, 120);        // N <= 128: 120 (measured in round 1)
  if (g.N <= 128) return (split || tiles(128) >= min_tiles128) ? launch_bn<128>(g, st) : launch_bn<64>(g, st);
  if (split || tiles(256) >= min_tiles) return launch_bn<256>(g, st);
  return tiles(128) >= min_tiles ? launch_bn<128>(g, st) : launch_bn<64>(g, st);
}

}  // namespace longer
