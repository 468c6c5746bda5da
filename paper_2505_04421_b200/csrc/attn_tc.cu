// attn_tc.cu — attention of the cross and self layers on the tensor cores (tcgen05), one CTA per
// (sample, head) — or per three samples in the self-layer backward.
//
// _multi_head_attention + masked_softmax (pkg/src/longrec/attention.py:153-169,
// pkg/src/longrec/tensors.py:323-351): the q = k + m query rows (≤ 128, zero-padded to the UMMA
// M = 128 tile) against the key rows (cross: v = G + m; self: the q rows themselves), streamed in
// chunks of 128 keys by 3-D TMA.  The structured visibility mask (VisRule) is one key interval per
// query row, evaluated in registers.
//
// Forward: one pass over the key chunks with a running max / sum per row and O += P̃·V in TMEM
// (rescaled in TMEM only when the max grows by more than kRescale); LSE and an fp32 copy of O are
// kept for the backward.
// Backward: pass 1 D_i = Σ_j P·dP; pass 2 per chunk S and dP = dO·Vᵀ in TMEM → dS = P ⊙ (dP − D) in
// smem → dV = Pᵀ·dO, dK = dSᵀ·Q (thread = key row on readout), dQ += dS·K accumulated in TMEM.
#include "fe_common.cuh"
#include "ops.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstdlib>

namespace longer {

using namespace fe;

namespace {

constexpr int kC = 128;     // keys per chunk

// thread `row` copies row `row` of a [rows x DH] bf16 matrix into a canonical K-major tile
template <int DH>
__device__ __forceinline__ void load_rows_bf16(bf16* tile, const bf16* src, int ld, int row, int nrows) {
#pragma unroll
  for (int c = 0; c < DH; c += 8) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < nrows) v = *reinterpret_cast<const uint4*>(src + (long long)row * ld + c);
    *reinterpret_cast<uint4*>(tile + canon(row, c, DH)) = v;
  }
}

// packed key row j = key j % nk of sample b0 + j / nk (zero past the P samples / the batch)
template <int DH>
__device__ __forceinline__ void load_key_packed(bf16* tile, const bf16* base, int ld, long long sb, int row, int nk,
                                                int b0, int pack, int B) {
  const int s = row / nk, j = row % nk;
  const bool ok = s < pack && b0 + s < B;
  const bf16* src = base + (long long)(b0 + s) * sb + (long long)j * ld;
#pragma unroll
  for (int c = 0; c < DH; c += 8) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (ok) v = *reinterpret_cast<const uint4*>(src + c);
    *reinterpret_cast<uint4*>(tile + canon(row, c, DH)) = v;
  }
}

// Query i sits in tile row qrow_of(i) = (i % 4)·32 + i / 4, so the q ≤ 128 queries of a sample are
// spread over all four TMEM lane quadrants (= all four worker warps) instead of crowding warp 0.
__device__ __forceinline__ int query_of_row(int row) { return (row & 31) * 4 + (row >> 5); }

// The visible keys of one query row form ONE interval [lo, hi) of the key index (VisRule; the query
// groups are sorted, so "key group ≤ query group" is "key index ≤ query index" in the self layers):
//   sequence query: non-pad sequence keys up to its own group (pad query: none);
//   global query of rank r: every non-pad sequence key, then the globals of rank ≤ r.
__device__ __forceinline__ void vis_interval(const VisRule& v, int i, int nk, int& lo, int& hi) {
  const int slo = v.self_keys ? v.jpad() : v.npg;          // first non-pad sequence key
  if (i < v.k) {
    if (v.qpad(i)) {
      lo = hi = 0;
      return;
    }
    lo = slo;
    hi = v.self_keys ? (v.learn ? v.k : i + 1) : v.qgroup(i) + 1;
  } else {
    lo = slo;
    hi = v.ns + (i - v.k) + 1;
  }
  hi = min(hi, nk);
  if (hi < lo) hi = lo;
}
// bit v set ⇔ key j0 + v ∈ [lo, hi)
__device__ __forceinline__ uint32_t vis_bits(int lo, int hi, int j0) {
  const int a = max(lo - j0, 0), b = min(hi - j0, 32);
  if (b <= a) return 0u;
  const uint32_t mb = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
  return mb & ~((1u << a) - 1u);
}

// Tile row r of a (sample, head) CTA ↔ its query: packed rows r % nq of sample b0 + r / nq, else
// query_of_row(r) of sample b0; false for rows past the queries / samples.
__device__ __forceinline__ bool tile_query(const AttnArgs& a, int b0, int pack, int r, int& b, int& qi) {
  const int sr = pack > 1 ? r / a.nq : 0;
  qi = pack > 1 ? r % a.nq : query_of_row(r);
  b = b0 + sr;
  return qi < a.nq && sr < pack && b < a.B;
}

// Forward, ONE pass over the key chunks: S = Q·K_cᵀ in TMEM; the workers keep a running max m
// and sum l per row and write P̃ = exp(s − m) (bf16) over the dead K tile; O += P̃·V_c accumulates
// in TMEM.  When a chunk raises a row's max by more than kRescale the row's O is rescaled in TMEM
// (tcgen05.ld/st) — rare after the first chunk; below that threshold P̃ ≤ e^kRescale stays exact
// enough in bf16 and fp32.  O/l, the fp32 copy and lse = m + log l are written at the end.
// Shared memory: Q + K|P + V (96 KB at head width 128) → two CTAs per SM.
constexpr float kRescale = 8.f;

// TMA (head width ≥ 64): K / V chunks arrive by 3-D TMA into 128-byte-swizzled tiles, the next
// chunk issued by the MMA thread as soon as O += P·V of the current one has completed.
// Packing (pack = P > 1, self layers): P samples share one CTA — tile row r is query r % nq of
// sample r / nq, key column j is key j % nk of sample j / nk (P·nq ≤ 128, P·nk ≤ 128: one chunk),
// and a row sees only its own sample's key interval, shifted by (r / nq)·nk.  K / V then come
// from a 2-D tensor map over the contiguous [B·nk] key rows.
// KVS (the cross layer with absorbed projections: keys and values are the same rows): one TMA tile
// per chunk serves as K (K-major, for S) and as V (MN-major, for P·V); P gets the K tile's slot.
template <int DH, bool TMA, bool KVS>
__global__ void __launch_bounds__(kThreads, 2) xattn_fwd_kernel(AttnArgs a, const __grid_constant__ CUtensorMap tmK,
                                                                 const __grid_constant__ CUtensorMap tmV, int pack) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int KP = kC * DH > 128 * kC ? kC * DH : 128 * kC;
  constexpr uint32_t TCOLS = DH > 128 ? 512 : 256;
  bf16* sQ = reinterpret_cast<bf16*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  bf16* sKP = sQ + 128 * DH;                      // K chunk (kC x DH), then P (128 x kC)
  bf16* sV = sKP + KP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kC * DH);
  uint64_t* bar_a = bars;
  uint64_t* bar_d = bars + 1;
  uint64_t* bar_kv = bars + 2;
  uint64_t* bar_m = bars + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int b0 = (blockIdx.x / a.heads) * pack, hd = blockIdx.x % a.heads;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_a, 32 * kWorkers);
    sm100::mbar_init(bar_d, 1);
    sm100::mbar_init(bar_kv, 1);
    sm100::mbar_init(bar_m, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<TCOLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  const uint32_t T_S = tmem, T_O = tmem + 128;
  const int nchunk = (a.nk + kC - 1) / kC;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t aQ = sm100::smem_u32(sQ), aKP = sm100::smem_u32(sKP), aV = sm100::smem_u32(sV);
      uint32_t pa = 0, pkv = 0, pm = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      auto load_kv = [&](int c) {
        sm100::mbar_arrive_expect_tx(bar_kv, (KVS ? 1 : 2) * kC * DH * 2);
#pragma unroll
        for (int i = 0; i < DH / 64; ++i) {
          if (pack > 1) {
            if (!KVS) sm100::tma_load_2d(sKP + i * kC * 64, &tmK, bar_kv, hd * DH + 64 * i, b0 * a.nk);
            sm100::tma_load_2d(sV + i * kC * 64, &tmV, bar_kv, hd * DH + 64 * i, b0 * a.nk);
          } else {
            if (!KVS) sm100::tma_load_3d(sKP + i * kC * 64, &tmK, bar_kv, hd * DH + 64 * i, c * kC, b0);
            sm100::tma_load_3d(sV + i * kC * 64, &tmV, bar_kv, hd * DH + 64 * i, c * kC, b0);
          }
        }
      };
      if constexpr (TMA) {
        sm100::tma_prefetch(&tmK);
        sm100::tma_prefetch(&tmV);
        load_kv(0);
      }
      for (int c = 0; c < nchunk; ++c) {
        wait_a();                                   // K_c, V_c staged (TMA: Q staged, TMEM S free)
        if constexpr (TMA) {
          sm100::mbar_wait(bar_kv, pkv);
          pkv ^= 1;
          mma(T_S, Opnd{aQ, DH, 0}, OpndSW{KVS ? aV : aKP, kC, 0}, DH / 16, kC, false);
        } else {
          mma(T_S, Opnd{aQ, DH, 0}, Opnd{aKP, DH, 0}, DH / 16, kC, false);
        }
        sm100::mma_commit(bar_d);
        wait_a();                                   // P_c staged (and O rescaled)
        if constexpr (TMA)
          mma(T_O, Opnd{aKP, kC, 0}, OpndSW{aV, kC, 1}, kC / 16, DH, c > 0);
        else
          mma(T_O, Opnd{aKP, kC, 0}, Opnd{aV, DH, 1}, kC / 16, DH, c > 0);
        sm100::mma_commit(bar_d);
        if constexpr (TMA) {
          if (c + 1 < nchunk) {                     // K|P and V free once O += P·V has completed
            sm100::mma_commit(bar_m);
            sm100::mbar_wait(bar_m, pm);
            pm ^= 1;
            load_kv(c + 1);
          }
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int sr = pack > 1 ? row / a.nq : 0;                  // packed sample of this row
    const int qi = pack > 1 ? row % a.nq : query_of_row(row);
    const int b = min(b0 + sr, a.B - 1);
    const uint32_t lo_lane = (uint32_t)(q * 32) << 16;
    const float scale = rsqrtf((float)(a.D / a.heads));
    const VisRule vis{a.k, a.G, a.ns, a.goff, a.npg[b], a.qg ? a.qg + (long long)b * a.k : nullptr, a.learn,
                     a.self_keys};
    const bool qrow = qi < a.nq && sr < pack && b0 + sr < a.B;
    int vlo = 0, vhi = 0;
    if (qrow) {
      vis_interval(vis, qi, a.nk, vlo, vhi);
      vlo += sr * a.nk;
      vhi += sr * a.nk;
    }
    const bf16* Qb = a.Q + b * a.sq + hd * DH;
    const bf16* Kb = a.Kp + b0 * a.sk + hd * DH;
    const bf16* Vb = a.V + b0 * a.sv + hd * DH;
    uint32_t pd = 0;
    auto signal = [&]() { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar_a); };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    (void)Qb;
    // the warp's 32 query rows into the canonical Q tile, cooperatively: 8 rows x 4 16-byte column
    // chunks per instruction (whole 64-byte row segments instead of 32 scattered pieces)
    {
      const int lr = lane & 7, kc = lane >> 3;
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        int bq, qq;
        const int r = q * 32 + rb * 8 + lr;
        const bool ok = tile_query(a, b0, pack, r, bq, qq);
        const bf16* src = a.Q + bq * a.sq + (long long)qq * a.ldq + hd * DH;
#pragma unroll
        for (int k = 0; k < DH / 32; ++k) {
          const int c = (4 * k + kc) * 8;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (ok) v = *reinterpret_cast<const uint4*>(src + c);
          *reinterpret_cast<uint4*>(sQ + canon(r, c, DH)) = v;
        }
      }
    }
    float m = -INFINITY, l = 0.f;
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * kC;
      if constexpr (!TMA) {
        if (pack > 1) {
          load_key_packed<DH>(sKP, a.Kp + hd * DH, a.ldk, a.sk, row, a.nk, b0, pack, a.B);
          load_key_packed<DH>(sV, a.V + hd * DH, a.ldv, a.sv, row, a.nk, b0, pack, a.B);
        } else {
          load_rows_bf16<DH>(sKP, Kb + (long long)c0 * a.ldk, a.ldk, row, a.nk - c0);
          load_rows_bf16<DH>(sV, Vb + (long long)c0 * a.ldv, a.ldv, row, a.nk - c0);
        }
      }
      signal();
      wait_d();                                     // S_c ready (K tile dead)
      float cm = -INFINITY;
#pragma unroll 1
      for (int j0 = 0; j0 < kC; j0 += 32) {
        float s[32];
        tmem_row<32>(T_S + lo_lane + j0, s);
        const uint32_t bits = vis_bits(vlo, vhi, c0 + j0);
        if (bits) {
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (bits & (1u << u)) cm = fmaxf(cm, s[u]);
        }
      }
      cm *= scale;
      const bool raise = cm > m + kRescale || (m == -INFINITY && cm != -INFINITY);
      float factor = 1.f;
      if (raise) {
        factor = m == -INFINITY ? 0.f : __expf(m - cm);
        l *= factor;
        m = cm;
      }
      if (c > 0 && __any_sync(0xffffffffu, raise)) {
#pragma unroll 1
        for (int cc = 0; cc < DH; cc += 32) {
          uint32_t r[32];
          sm100::tmem_ld32(T_O + lo_lane + cc, r);
          sm100::tmem_ld_wait();
          sm100::reg_fence(r);
#pragma unroll
          for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * factor);
          sm100::tmem_st32(T_O + lo_lane + cc, r);
        }
        sm100::tmem_st_wait();
      }
#pragma unroll 1
      for (int j0 = 0; j0 < kC; j0 += 32) {
        float s[32];
        tmem_row<32>(T_S + lo_lane + j0, s);
        const uint32_t bits = vis_bits(vlo, vhi, c0 + j0);
        float add = 0.f;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          s[u] = (bits & (1u << u)) ? __expf(fmaf(s[u], scale, -m)) : 0.f;
          add += s[u];
        }
        l += add;
        store_row(sKP, row, kC, s, 32, j0);
      }
      signal();
      wait_d();                                     // O += P·V done: K|P and V tiles free
    }
    const float rl = l > 0.f ? 1.f / l : 0.f;
    // O / l as bf16 rows through this warp's quarter of the (free: the last P·V is done) K|P tile,
    // XOR-swizzled 16-byte chunks, out as whole rows; the fp32 copy (the SIMT backward's D_i input)
    // only when asked for
    constexpr int CH = DH / 8;                            // 16-byte chunks per bf16 row
    constexpr int XM = CH >= 8 ? 7 : CH - 1;              // swizzle mask
    uint4* stg = reinterpret_cast<uint4*>(sKP) + q * 32 * CH;
    float* dst32 = a.ctx32 ? a.ctx32 + b * a.sc + (long long)qi * a.ldc + hd * DH : nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < DH; c0 += 32) {
      float o[32];
      tmem_row<32>(T_O + lo_lane + c0, o);
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        float w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = o[c + u] * rl;
        const int j = (c0 + c) / 8;
        stg[lane * CH + (j ^ (lane & XM))] = make_uint4(sm100::pack_bf16(w[0], w[1]), sm100::pack_bf16(w[2], w[3]),
                                                       sm100::pack_bf16(w[4], w[5]), sm100::pack_bf16(w[6], w[7]));
        if (dst32 && qrow) {
          *reinterpret_cast<float4*>(dst32 + c0 + c) = make_float4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<float4*>(dst32 + c0 + c + 4) = make_float4(w[4], w[5], w[6], w[7]);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int idx = k * 32 + lane, r = idx / CH, sg = idx % CH;
      int bq, qq;
      if (tile_query(a, b0, pack, q * 32 + r, bq, qq))
        *reinterpret_cast<uint4*>(a.ctx + bq * a.sc + (long long)qq * a.ldc + hd * DH + sg * 8) =
            stg[r * CH + (sg ^ (r & XM))];
    }
    if (qrow) a.lse[((long long)b * a.heads + hd) * a.nq + qi] = l > 0.f ? m + __logf(l) : -INFINITY;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<TCOLS>(tmem);
}

// Head width 256 (BIG): the 512 TMEM columns hold S|dV-half, dP|dK-half and dQ (256); dV and dK come
// out in two 128-column halves.  Shared memory keeps only QR = 64 query rows of Q, dO, P and dS
// (nq ≤ 64, identity row order): the M = 128 MMAs read rows 64..127 from the next buffer and
// produce rows that are never read, and the K = query contractions stop at 64.
// Eight worker warps, two per TMEM lane quadrant: the pair shares its 32 rows and splits the
// columns (key columns of S / dP, head columns of the loads and the dV / dK / dQ read-outs); the
// row sums D_i meet once in shared memory after pass 1.
// TMA (head width ≥ 64): the MMA thread streams each K / V chunk with 3-D tensor maps ([sample]
// [key][column], rows past the sample's keys read as zero) into 128-byte-swizzled tiles, issuing
// the next chunk as soon as the MMAs reading the current one have completed.
// Packing as in the forward (pack > 1: non-BIG only; key rows of dV / dK map back to their samples).
// SHORT (head width ≤ 128, one sample per CTA with nq ≤ 64 — the cross layer): the 64-row query
// tiles of BIG free 64 KB of shared memory for a second K / V buffer, so the TMA of chunk i+2 is in
// flight while chunk i+1 is computed (the chunk sequence is pass 1 then pass 2), and the dV / dK
// rows leave through a per-warp shared-memory transpose as 64-byte row segments.
// KVS (with SHORT; keys = values, the absorbed cross layer): one TMA tile per chunk serves K and V
// (32 KB buffers), and dV + dK accumulate into one TMEM region (Pᵀ·dO then += dSᵀ·Q).
template <int DH, bool TMA, bool SHORT, bool KVS>
__global__ void __launch_bounds__(kThreads8, 1) xattn_bwd_kernel(AttnArgs a, const __grid_constant__ CUtensorMap tmK,
                                                                  const __grid_constant__ CUtensorMap tmV, int pack) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr bool BIG = DH > 128;
  static_assert(!SHORT || (TMA && !BIG), "SHORT: TMA path at head width <= 128");
  static_assert(!KVS || SHORT, "KVS: with SHORT");
  constexpr int KVT = KVS ? 1 : 2;                // tiles per K / V buffer
  constexpr int QR = (BIG || SHORT) ? 64 : 128;   // stored query rows
  constexpr int KVB = SHORT ? 2 : 1;              // K / V buffers
  bf16* sQ = reinterpret_cast<bf16*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  bf16* sdO = sQ + QR * DH;
  bf16* sK = sdO + QR * DH;                       // buffer b: K at sK + b·KVT·kC·DH, V right after it
  bf16* sV = sK + kC * DH;
  bf16* sdS = sK + KVB * KVT * kC * DH;           // QR x kC  (pre-scaled by 1/sqrt(dh))
  bf16* sP = sdS + QR * kC;                       // QR x kC  (after dS: dS's M-row overread stays in smem)
  float* sDp = reinterpret_cast<float*>(sP + QR * kC);       // [2][128] partial D_i of the two groups
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDp + 256);
  uint64_t* bar_a = bars;
  uint64_t* bar_d = bars + 1;
  uint64_t* bar_m = bars + 2;                     // TMA: the MMAs reading a chunk are done
  uint64_t* bar_kv = bars + 3;                    // [KVB] TMA: K / V chunk landed in buffer b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 + KVB);
  const int b0 = (blockIdx.x / a.heads) * pack, hd = blockIdx.x % a.heads;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_a, 32 * 2 * kWorkers);
    sm100::mbar_init(bar_d, 1);
    for (int b = 0; b < KVB; ++b) sm100::mbar_init(&bar_kv[b], 1);
    sm100::mbar_init(bar_m, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  const uint32_t T_A = tmem, T_B = tmem + 128, T_DQ = tmem + 256;
  const int nchunk = (a.nk + kC - 1) / kC;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t aQ = sm100::smem_u32(sQ), adO = sm100::smem_u32(sdO), aK0 = sm100::smem_u32(sK);
      const uint32_t aP = sm100::smem_u32(sP), adS = sm100::smem_u32(sdS);
      constexpr uint32_t kBufBytes = KVT * kC * DH * 2;
      uint32_t pa = 0, pkv0 = 0, pkv1 = 0, pm = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      // the chunk sequence: pass 1 over chunks 0..n-1, then (n > 1) pass 2 over them again; load i
      // goes to buffer i % KVB
      const int nload = nchunk > 1 ? 2 * nchunk : 1;
      auto load_kv = [&](int i) {
        const int c = i % nchunk, bsel = i % KVB;
        bf16* dK = sK + bsel * KVT * kC * DH;
        bf16* dV = dK + kC * DH;
        sm100::mbar_arrive_expect_tx(&bar_kv[bsel], KVT * kC * DH * 2);
#pragma unroll
        for (int i2 = 0; i2 < DH / 64; ++i2) {
          if (pack > 1) {
            sm100::tma_load_2d(dK + i2 * kC * 64, &tmK, &bar_kv[bsel], hd * DH + 64 * i2, b0 * a.nk);
            if (!KVS) sm100::tma_load_2d(dV + i2 * kC * 64, &tmV, &bar_kv[bsel], hd * DH + 64 * i2, b0 * a.nk);
          } else {
            sm100::tma_load_3d(dK + i2 * kC * 64, &tmK, &bar_kv[bsel], hd * DH + 64 * i2, c * kC, b0);
            if (!KVS) sm100::tma_load_3d(dV + i2 * kC * 64, &tmV, &bar_kv[bsel], hd * DH + 64 * i2, c * kC, b0);
          }
        }
      };
      auto wait_kv = [&](int i) {
        if (i % KVB == 0) { sm100::mbar_wait(&bar_kv[0], pkv0); pkv0 ^= 1; }
        else { sm100::mbar_wait(&bar_kv[KVB - 1], pkv1); pkv1 ^= 1; }
      };
      auto mma_done = [&]() { sm100::mma_commit(bar_m); sm100::mbar_wait(bar_m, pm); pm ^= 1; };
      // once the MMAs reading load i are done, its buffer takes load i + KVB
      auto refill = [&](int i) {
        if (i + KVB < nload) { mma_done(); load_kv(i + KVB); }
      };
      auto kaddr = [&](int i) { return aK0 + (uint32_t)(i % KVB) * kBufBytes; };
      // S = Q·Kᵀ and dP = dO·Vᵀ of the chunk of load i
      auto mma_s_dp = [&](int i) {
        const uint32_t aK = kaddr(i), aV = KVS ? aK : aK + kC * DH * 2;
        if constexpr (TMA) {
          mma(T_A, Opnd{aQ, DH, 0}, OpndSW{aK, kC, 0}, DH / 16, kC, false);
          mma(T_B, Opnd{adO, DH, 0}, OpndSW{aV, kC, 0}, DH / 16, kC, false);
        } else {
          mma(T_A, Opnd{aQ, DH, 0}, Opnd{aK, DH, 0}, DH / 16, kC, false);
          mma(T_B, Opnd{adO, DH, 0}, Opnd{aV, DH, 0}, DH / 16, kC, false);
        }
      };
      if constexpr (TMA) {
        sm100::tma_prefetch(&tmK);
        sm100::tma_prefetch(&tmV);
        for (int i = 0; i < KVB && i < nload; ++i) load_kv(i);
      }
      for (int c = 0; c < nchunk; ++c) {                            // pass 1: D = Σ_j P·dP
        wait_a();
        if constexpr (TMA) wait_kv(c);
        mma_s_dp(c);
        sm100::mma_commit(bar_d);
        if constexpr (TMA) refill(c);
      }
      constexpr int NH = BIG ? 2 : 1, NW = DH / NH;                // dV / dK column halves
      for (int c = 0; c < nchunk; ++c) {
        const int i = nchunk > 1 ? nchunk + c : 0;                  // load index of this chunk
        if (nchunk > 1) {           // a single chunk's S and dP are still in TMEM from pass 1
          wait_a();                                                 // K, V chunk (+ Q, dO)
          if constexpr (TMA) wait_kv(i);
          mma_s_dp(i);
          sm100::mma_commit(bar_d);
        }
        const uint32_t aK = kaddr(i);
        for (int h = 0; h < NH; ++h) {
          wait_a();                                                 // P, dS (h = 1: halves read out)
          const uint32_t co = (uint32_t)h * NW * 16;                // byte offset of column half h
          mma(T_A, Opnd{aP, kC, 1}, Opnd{adO + co, DH, 1}, QR / 16, NW, false);   // dV = Pᵀ·dO
          mma(KVS ? T_A : T_B, Opnd{adS, kC, 1}, Opnd{aQ + co, DH, 1}, QR / 16, NW, KVS);   // dK = dSᵀ·Q
          if (h == 0)
            for (int hq = 0; hq < NH; ++hq) {                                      // dQ += dS·K
              if constexpr (TMA)
                mma(T_DQ + hq * NW, Opnd{adS, kC, 0}, OpndSW{aK + (uint32_t)hq * (NW / 64) * kC * 128, kC, 1},
                    kC / 16, NW, c > 0);
              else
                mma(T_DQ + hq * NW, Opnd{adS, kC, 0}, Opnd{aK + (uint32_t)hq * NW * 16, DH, 1}, kC / 16, NW, c > 0);
            }
          sm100::mma_commit(bar_d);
        }
        if constexpr (TMA) {
          if (nchunk > 1) refill(i);
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int grp = (warp - 1) >> 2;                 // column half of this warp pair
    const int row = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    constexpr int HC = DH / 2;                       // head columns per group
    // read-out columns (32 at a time) of this group for dV / dK (per half) and dQ; at DH = 32 the
    // first group reads all of them
    constexpr int RW = BIG ? DH / 4 : (DH >= 64 ? DH / 2 : DH);       // dV / dK (per half)
    const int r0 = DH >= 64 ? grp * RW : 0, r1 = DH >= 64 ? r0 + RW : (grp == 0 ? DH : 0);
    const int q0 = DH >= 64 ? grp * HC : 0, q1 = DH >= 64 ? q0 + HC : (grp == 0 ? DH : 0);   // dQ
    const float scale = rsqrtf((float)(a.D / a.heads));
    const int sr = pack > 1 ? row / a.nq : 0;                  // packed sample of this query row
    const int b = min(b0 + sr, a.B - 1);
    const VisRule vis{a.k, a.G, a.ns, a.goff, a.npg[b], a.qg ? a.qg + (long long)b * a.k : nullptr, a.learn,
                     a.self_keys};
    const bf16* Qb = a.Q + b * a.sq + hd * DH;
    const bf16* Kb = a.Kp + b0 * a.sk + hd * DH;
    const bf16* Vb = a.V + b0 * a.sv + hd * DH;
    uint32_t pd = 0;
    auto signal = [&]() { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar_a); };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    // this group's half of a K / V chunk: key row `row`, head columns [grp·HC, grp·HC + HC)
    auto load_half = [&](bf16* tile, const bf16* src, int ld, int nrows) {
#pragma unroll
      for (int c = 0; c < HC; c += 8) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row < nrows) v = *reinterpret_cast<const uint4*>(src + (long long)row * ld + grp * HC + c);
        *reinterpret_cast<uint4*>(tile + canon(row, grp * HC + c, DH)) = v;
      }
    };
    const int qi = pack > 1 ? row % a.nq : ((BIG || SHORT) ? row : query_of_row(row));
    const bool qrow = qi < a.nq && sr < pack && b0 + sr < a.B;
    if (QR == 128 || row < QR) {
#pragma unroll
      for (int c = grp * HC; c < grp * HC + HC; c += 8) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (qrow) v = *reinterpret_cast<const uint4*>(Qb + (long long)qi * a.ldq + c);
        *reinterpret_cast<uint4*>(sQ + canon(row, c, DH)) = v;
      }
    }
    // dO (fp32) → bf16 tile
    float Di = 0.f, lse = -INFINITY;
    {
      const float* dOr = a.dctx + b * a.sdc + (long long)qi * a.lddc + hd * DH;
#pragma unroll
      for (int c = grp * HC; c < grp * HC + HC; c += 8) {
        if (QR < 128 && row >= QR) break;
        float v[8];
        if (qrow) {
          const float4 x = *reinterpret_cast<const float4*>(dOr + c), y = *reinterpret_cast<const float4*>(dOr + c + 4);
          v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = 0.f;
        }
        store_row(sdO, row, DH, v, 8, c);
      }
      if (qrow) lse = a.lse[((long long)b * a.heads + hd) * a.nq + qi];
    }
    int vlo = 0, vhi = 0;
    if (qrow && lse != -INFINITY) {
      vis_interval(vis, qi, a.nk, vlo, vhi);
      vlo += sr * a.nk;
      vhi += sr * a.nk;
    }
    // this group's half of the packed key row `row` (pack > 1)
    auto load_half_packed = [&](bf16* tile, const bf16* base, int ld, long long sb) {
      const int s2 = row / a.nk, j = row % a.nk;
      const bool ok = s2 < pack && b0 + s2 < a.B;
      const bf16* src = base + (long long)(b0 + s2) * sb + (long long)j * ld + hd * DH;
#pragma unroll
      for (int c = 0; c < HC; c += 8) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ok) v = *reinterpret_cast<const uint4*>(src + grp * HC + c);
        *reinterpret_cast<uint4*>(tile + canon(row, grp * HC + c, DH)) = v;
      }
    };
    // pass 1: D_i = Σ_j P_ij dP_ij with exactly the P and dP of pass 2, so that Σ_j dS_ij = 0
    // holds to rounding (D = rowsum(dO ⊙ O) would mix the bf16 roundings of dO, P and V).
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * kC;
      if constexpr (!TMA) {
        if (pack > 1) {
          load_half_packed(sK, a.Kp, a.ldk, a.sk);
          load_half_packed(sV, a.V, a.ldv, a.sv);
        } else {
          load_half(sK, Kb + (long long)c0 * a.ldk, a.ldk, a.nk - c0);
          load_half(sV, Vb + (long long)c0 * a.ldv, a.ldv, a.nk - c0);
        }
      }
      signal();
      wait_d();
#pragma unroll 1
      for (int j0 = grp * (kC / 2); j0 < grp * (kC / 2) + kC / 2; j0 += 32) {
        float s[32], dp[32];
        tmem_row2<32>(T_A + lo + j0, s, T_B + lo + j0, dp);
        const uint32_t bits = vis_bits(vlo, vhi, c0 + j0);
        if (bits) {
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (bits & (1u << u)) Di = fmaf(__expf(fmaf(s[u], scale, -lse)), dp[u], Di);
        }
      }
    }
    sDp[grp * 128 + row] = Di;                       // combine the two column halves of D_i
    asm volatile("bar.sync 1, 256;" ::: "memory");
    Di = sDp[row] + sDp[128 + row];
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * kC;
      if (nchunk > 1) {                 // a single chunk (K, V, S, dP) is still resident from pass 1
        if constexpr (!TMA) {
          load_half(sK, Kb + (long long)c0 * a.ldk, a.ldk, a.nk - c0);
          load_half(sV, Vb + (long long)c0 * a.ldv, a.ldv, a.nk - c0);
        }
        signal();
        wait_d();
      }
#pragma unroll 1
      for (int j0 = grp * (kC / 2); j0 < grp * (kC / 2) + kC / 2; j0 += 32) {
        float s[32], dp[32];
        tmem_row2<32>(T_A + lo + j0, s, T_B + lo + j0, dp);
        const uint32_t bits = vis_bits(vlo, vhi, c0 + j0);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const float p = (bits & (1u << u)) ? __expf(fmaf(s[u], scale, -lse)) : 0.f;
          s[u] = p;
          dp[u] = p * (dp[u] - Di) * scale;
        }
        if (QR == 128 || row < QR) {
          store_row(sP, row, kC, s, 32, j0);
          store_row(sdS, row, kC, dp, 32, j0);
        }
      }
      // thread = key row: dV, dK of key c0 + row, 32 columns at a time (BIG: two 128-column halves)
      // key row → (sample, key): packed rows map back to their own sample
      const int ks = pack > 1 ? row / a.nk : 0, kj = pack > 1 ? row % a.nk : c0 + row;
      const bool krow = pack > 1 ? (ks < pack && b0 + ks < a.B) : (c0 + row < a.nk);
      bf16* pv = a.dV + (long long)(b0 + ks) * a.sdv + (long long)kj * a.lddv + hd * DH;
      bf16* pk = a.dK + (long long)(b0 + ks) * a.sdk + (long long)kj * a.lddk + hd * DH;
      constexpr int NH = BIG ? 2 : 1, NW = DH / NH;
      for (int h = 0; h < NH; ++h) {
        signal();
        wait_d();
#pragma unroll 1
        for (int c1 = r0; c1 < r1; c1 += 32) {
          float dv[32], dk[32];
          if constexpr (KVS) {                  // T_A holds dV + dK
            tmem_row<32>(T_A + lo + c1, dk);
#pragma unroll
            for (int u = 0; u < 32; ++u) dv[u] = 0.f;
          } else {
            tmem_row2<32>(T_A + lo + c1, dv, T_B + lo + c1, dk);
          }
          if constexpr (SHORT) {
            // through this warp's 2 × 2 KB of the (consumed) dS / P tiles: 16-byte segments
            // XOR-swizzled, conflict-free both ways; out as 64-byte row segments
            uint4* stg = reinterpret_cast<uint4*>(sdS) + (warp - 1) * 256;
            if (a.sum_kv && !KVS) {
#pragma unroll
              for (int u = 0; u < 32; ++u) dk[u] += dv[u];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int sl = lane * 4 + (j ^ ((lane >> 1) & 3));
              stg[sl] = make_uint4(sm100::pack_bf16(dv[8 * j], dv[8 * j + 1]), sm100::pack_bf16(dv[8 * j + 2], dv[8 * j + 3]),
                                   sm100::pack_bf16(dv[8 * j + 4], dv[8 * j + 5]), sm100::pack_bf16(dv[8 * j + 6], dv[8 * j + 7]));
              stg[128 + sl] = make_uint4(sm100::pack_bf16(dk[8 * j], dk[8 * j + 1]), sm100::pack_bf16(dk[8 * j + 2], dk[8 * j + 3]),
                                         sm100::pack_bf16(dk[8 * j + 4], dk[8 * j + 5]), sm100::pack_bf16(dk[8 * j + 6], dk[8 * j + 7]));
            }
            __syncwarp();
            const int kbase = c0 + q * 32;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int r = k * 8 + (lane >> 2), sgm = lane & 3;
              if (kbase + r < a.nk) {
                const long long off = (long long)(kbase + r);
                const int sl = r * 4 + (sgm ^ ((r >> 1) & 3));
                if (!a.sum_kv)
                  *reinterpret_cast<uint4*>(a.dV + (long long)b0 * a.sdv + off * a.lddv + hd * DH + c1 + sgm * 8) = stg[sl];
                *reinterpret_cast<uint4*>(a.dK + (long long)b0 * a.sdk + off * a.lddk + hd * DH + c1 + sgm * 8) = stg[128 + sl];
              }
            }
            __syncwarp();
            continue;
          }
          if (!krow) continue;
          if (a.sum_kv) {
#pragma unroll
            for (int u = 0; u < 32; ++u) dk[u] += dv[u];
          }
#pragma unroll
          for (int cc = 0; cc < 32; cc += 8) {
            uint4 x, y;
            x.x = sm100::pack_bf16(dv[cc], dv[cc + 1]); x.y = sm100::pack_bf16(dv[cc + 2], dv[cc + 3]);
            x.z = sm100::pack_bf16(dv[cc + 4], dv[cc + 5]); x.w = sm100::pack_bf16(dv[cc + 6], dv[cc + 7]);
            y.x = sm100::pack_bf16(dk[cc], dk[cc + 1]); y.y = sm100::pack_bf16(dk[cc + 2], dk[cc + 3]);
            y.z = sm100::pack_bf16(dk[cc + 4], dk[cc + 5]); y.w = sm100::pack_bf16(dk[cc + 6], dk[cc + 7]);
            if (!a.sum_kv) *reinterpret_cast<uint4*>(pv + h * NW + c1 + cc) = x;
            *reinterpret_cast<uint4*>(pk + h * NW + c1 + cc) = y;
          }
        }
      }
    }
    bf16* pq = a.dQ + b * a.sdq + (long long)qi * a.lddq + hd * DH;
#pragma unroll 1
    for (int c0 = q0; c0 < q1; c0 += 32) {
      float dq[32];
      tmem_row<32>(T_DQ + lo + c0, dq);
      if (!qrow) continue;
#pragma unroll
      for (int cc = 0; cc < 32; cc += 8) {
        uint4 x;
        x.x = sm100::pack_bf16(dq[cc], dq[cc + 1]); x.y = sm100::pack_bf16(dq[cc + 2], dq[cc + 3]);
        x.z = sm100::pack_bf16(dq[cc + 4], dq[cc + 5]); x.w = sm100::pack_bf16(dq[cc + 6], dq[cc + 7]);
        *reinterpret_cast<uint4*>(pq + c0 + cc) = x;
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ transposed backward (keys = values)
// The absorbed cross layer's backward (one sample per CTA, nq ≤ 64 queries, nk keys = values = kn)
// with the KEYS as the tile rows: Sᵀ = K·Q'ᵀ and dPᵀ = K·dOᵀ land as [128 keys × 64 queries] in
// TMEM, double-buffered, so the tensor core computes chunk i+1 while the workers turn chunk i into
// Pᵀ and dSᵀ — and every lane of every worker warp is a key row (in the query-row layout only the
// 35 query rows of 128 lanes had work).  The chunk sequence is pass 1 then pass 2 (K tiles by 3-D
// TMA, two buffers, the refill of one issued while the other is computed).
//   pass 1: D_q = Σ_k P_kq·dP_kq (per-thread sums over the chunks, a warp column sum, a 4-quarter
//           reduction in shared memory) — with exactly the P and dP of pass 2, so Σ_k dS_kq = 0;
//   pass 2: Pᵀ, dSᵀ = Pᵀ ⊙ (dPᵀ − D)·scale → shared memory → dKV = Pᵀ·dO + dSᵀ·Q' (one TMEM
//           accumulator: keys are values) and dQ' += dS·K (dS read MN-major from the dSᵀ tile).
// TMEM: Sᵀ ×2, dPᵀ ×2 (64 columns each), dKV (DH), dQ' (DH) = 512 columns at DH = 128.
template <int DH>
__global__ void __launch_bounds__(kThreads8, 1) xattn_bwd_t_kernel(AttnArgs a, const __grid_constant__ CUtensorMap tmK) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int NQ = 64, PT = 128;                // query columns; P / dS tile row length (zero-padded)
  bf16* sK = reinterpret_cast<bf16*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  bf16* sQ = sK + 2 * kC * DH;                    // NQ x DH  Q'  (canonical K-major)
  bf16* sdO = sQ + NQ * DH;                       // NQ x DH  dO
  bf16* sPT = sdO + NQ * DH;                      // kC x PT  Pᵀ  (keys x queries)
  bf16* sdST = sPT + kC * PT;                     // kC x PT  dSᵀ
  uint4* sStg = reinterpret_cast<uint4*>(sdST + kC * PT);      // per worker warp: 32 x 32 bf16
  float* sL = reinterpret_cast<float*>(sStg + 8 * 128);        // lse [NQ]
  float* sD = sL + NQ;                                         // D [NQ]
  float* sDp = sD + NQ;                                        // [4][NQ] per-quarter partial D
  int* sVlo = reinterpret_cast<int*>(sDp + 4 * NQ);            // visible key interval per query
  int* sVhi = sVlo + NQ;
  int* sMono = sVhi + NQ;                                      // [2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMono + 2);
  uint64_t* bar_kv = bars;            // [2] K tile landed
  uint64_t* bar_sd = bars + 2;        // [2] Sᵀ / dPᵀ buffer ready
  uint64_t* bar_fr = bars + 4;        // [2] Sᵀ / dPᵀ buffer read out by the workers
  uint64_t* bar_kf = bars + 6;        // [2] the MMAs reading K buffer b are done
  uint64_t* bar_pd = bars + 8;        // Pᵀ / dSᵀ written
  uint64_t* bar_kvd = bars + 9;       // dKV / dQ' MMAs done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  const int b = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) sm100::mbar_init(&bars[i], (i >= 4 && i < 6) ? 32 * 2 * kWorkers : 1);
    sm100::mbar_init(bar_pd, 32 * 2 * kWorkers);
    sm100::mbar_init(bar_kvd, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<512>(tmem_slot);
  pdl_trigger();
  pdl_wait();
  // operand tiles and per-query tables (every thread)
  const float scale = rsqrtf((float)a.D);
  const int nq = a.nq;
  for (int e = threadIdx.x; e < NQ * DH / 8; e += blockDim.x) {
    const int r = e / (DH / 8), c = (e % (DH / 8)) * 8;
    uint4 qv = make_uint4(0, 0, 0, 0), ov = qv;
    if (r < nq) {
      qv = *reinterpret_cast<const uint4*>(a.Q + b * a.sq + (long long)r * a.ldq + c);
      const float* src = a.dctx + b * a.sdc + (long long)r * a.lddc + c;
      const float4 x = *reinterpret_cast<const float4*>(src), y = *reinterpret_cast<const float4*>(src + 4);
      ov = make_uint4(sm100::pack_bf16(x.x, x.y), sm100::pack_bf16(x.z, x.w), sm100::pack_bf16(y.x, y.y),
                      sm100::pack_bf16(y.z, y.w));
    }
    *reinterpret_cast<uint4*>(sQ + canon(r, c, DH)) = qv;
    *reinterpret_cast<uint4*>(sdO + canon(r, c, DH)) = ov;
  }
  for (int e = threadIdx.x; e < 2 * kC * PT / 8; e += blockDim.x) reinterpret_cast<uint4*>(sPT)[e] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < NQ) {
    const int qi = threadIdx.x;
    int lo = 0, hi = 0;
    float lse = 0.f;
    if (qi < nq) {
      const VisRule vis{a.k, a.G, a.ns, a.goff, a.npg[b], a.qg ? a.qg + (long long)b * a.k : nullptr, a.learn,
                       a.self_keys};
      lse = a.lse[(long long)b * nq + qi];
      if (lse != -INFINITY) vis_interval(vis, qi, a.nk, lo, hi);
    }
    sVlo[qi] = lo; sVhi[qi] = hi; sL[qi] = lse;
  }
  // Cross-layer intervals share one lower end (the first non-pad key) and their upper ends never
  // decrease with the query index (sorted query groups, then the globals by rank; pad queries
  // first with an empty interval): a key row's visible columns are then a suffix of the valid
  // queries, found by a binary search instead of a test per column.  Verified here.
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1, lo0 = -1;
    for (int qi = 0; qi < nq; ++qi) {
      if (qi > 0 && sVhi[qi] < sVhi[qi - 1]) ok = 0;
      if (sVhi[qi] > sVlo[qi]) {
        if (lo0 < 0) lo0 = sVlo[qi];
        else if (sVlo[qi] != lo0) ok = 0;
      } else if (sVhi[qi] != 0) ok = 0;
    }
    sMono[0] = ok ? (lo0 < 0 ? (1 << 30) : lo0) : -1;   // the shared lower end, or -1: test per column
  }
  sm100::fence_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t T_KV = tmem + 256, T_Q = tmem + 256 + DH;
  auto T_S = [&](int sb) { return tmem + 64 * sb; };
  auto T_P = [&](int sb) { return tmem + 128 + 64 * sb; };
  const int nchunk = (a.nk + kC - 1) / kC;
  const int nload = 2 * nchunk;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t aK0 = sm100::smem_u32(sK), aQ = sm100::smem_u32(sQ), adO = sm100::smem_u32(sdO);
      const uint32_t aPT = sm100::smem_u32(sPT), adST = sm100::smem_u32(sdST);
      constexpr uint32_t kBuf = kC * DH * 2;
      uint32_t kvph = 0, frph = 0, kfph = 0, pdph = 0;     // parity bits: bit b = buffer b
      auto load = [&](int i) {
        const int kb = i & 1;
        bf16* dst = sK + kb * kC * DH;
        sm100::mbar_arrive_expect_tx(&bar_kv[kb], kC * DH * 2);
#pragma unroll
        for (int i2 = 0; i2 < DH / 64; ++i2)
          sm100::tma_load_3d(dst + i2 * kC * 64, &tmK, &bar_kv[kb], 64 * i2, (i % nchunk) * kC, b);
      };
      auto wait_bit = [&](uint64_t* bar, uint32_t& ph, int bit) {
        sm100::mbar_wait(bar, (ph >> bit) & 1u);
        ph ^= 1u << bit;
      };
      // Sᵀ / dPᵀ of load i into buffer i & 1 (its K tile landed; the workers read out use i-2)
      auto issue_sd = [&](int i) {
        const int kb = i & 1;
        wait_bit(&bar_kv[kb], kvph, kb);
        if (i >= 2) wait_bit(&bar_fr[kb], frph, kb);
        sm100::tc_fence_after();
        const uint32_t aK = aK0 + kb * kBuf;
        mma(T_S(kb), OpndSW{aK, kC, 0}, Opnd{aQ, DH, 0}, DH / 16, NQ, false);       // Sᵀ  = K·Q'ᵀ
        mma(T_P(kb), OpndSW{aK, kC, 0}, Opnd{adO, DH, 0}, DH / 16, NQ, false);      // dPᵀ = K·dOᵀ
        sm100::mma_commit(&bar_sd[kb]);
      };
      sm100::tma_prefetch(&tmK);
      load(0);
      if (nload > 1) load(1);
      issue_sd(0);
      for (int i = 0; i < nload; ++i) {
        const int kb = i & 1;
        // the next chunk's scores first: the tensor core works on them while the workers turn
        // this chunk into Pᵀ / dSᵀ
        if (i + 1 < nload) issue_sd(i + 1);
        if (i >= nchunk) {
          sm100::mbar_wait(bar_pd, pdph);
          pdph ^= 1;
          sm100::tc_fence_after();
          const uint32_t aK = aK0 + kb * kBuf;
          mma(T_KV, Opnd{aPT, PT, 0}, Opnd{adO, DH, 1}, NQ / 16, DH, false);        // Pᵀ·dO
          mma(T_KV, Opnd{adST, PT, 0}, Opnd{aQ, DH, 1}, NQ / 16, DH, true);         // + dSᵀ·Q'
          mma(T_Q, Opnd{adST, PT, 1}, OpndSW{aK, kC, 1}, kC / 16, DH, i > nchunk);   // dQ' += dS·K
          sm100::mma_commit(bar_kvd);
        }
        if (i + 2 < nload) {                            // K buffer kb: refill once use i is done
          sm100::mma_commit(&bar_kf[kb]);
          wait_bit(&bar_kf[kb], kfph, kb);
          load(i + 2);
        }
      }
    }
  } else {
    const int q = warp & 3, g = (warp - 1) >> 2;
    const int row = q * 32 + lane;                    // key row within a chunk (= TMEM lane)
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const int c0 = 32 * g;                            // this warp's query columns
    uint32_t sdph = 0, kvdph = 0;
    auto signal = [&](uint64_t* bar) { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar); };
    auto load_sd = [&](int i, float (&s)[32], float (&dp)[32]) {
      const int sb = i & 1;
      sm100::mbar_wait(&bar_sd[sb], (sdph >> sb) & 1u);
      sdph ^= 1u << sb;
      sm100::tc_fence_after();
      tmem_row2<32>(T_S(sb) + lo + c0, s, T_P(sb) + lo + c0, dp);
      sm100::tc_fence_before();
      sm100::mbar_arrive(&bar_fr[sb]);
    };
    // visible columns [c0, c0 + 32) of key row `key`, bit u = column c0 + u
    const int mono = sMono[0];
    auto vis_mask = [&](int key) -> uint32_t {
      if (mono >= 0) {
        if (key < mono) return 0u;
        int lo_c = c0, hi_c = min(c0 + 32, nq);       // first column with vhi > key (vhi sorted)
        while (lo_c < hi_c) {
          const int mid = (lo_c + hi_c) >> 1;
          if (sVhi[mid] > key) hi_c = mid; else lo_c = mid + 1;
        }
        const int end = min(c0 + 32, nq);
        if (lo_c >= end) return 0u;
        const uint32_t from = lo_c - c0, to = end - c0;   // bits [from, to)
        return (to >= 32 ? 0xffffffffu : ((1u << to) - 1u)) & ~((1u << from) - 1u);
      }
      uint32_t m = 0;
#pragma unroll
      for (int u = 0; u < 32; ++u) m |= (key >= sVlo[c0 + u] && key < sVhi[c0 + u]) ? (1u << u) : 0u;
      return m;
    };
    // pass 1: D
    {
      float dacc[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) dacc[u] = 0.f;
      for (int i = 0; i < nchunk; ++i) {
        float s[32], dp[32];
        load_sd(i, s, dp);
        const uint32_t m = vis_mask(i * kC + row);
        if (m) {
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (m & (1u << u)) dacc[u] = fmaf(__expf(fmaf(s[u], scale, -sL[c0 + u])), dp[u], dacc[u]);
        }
      }
      const float col = warp_colsum<32>(dacc);       // lane l: column c0 + l over this warp's rows
      sDp[q * NQ + c0 + lane] = col;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x - 32 < NQ) {
        const int cc = threadIdx.x - 32;
        sD[cc] = (sDp[cc] + sDp[NQ + cc]) + (sDp[2 * NQ + cc] + sDp[3 * NQ + cc]);
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    // dKV rows of chunk c: read out of TMEM as bf16 pairs (so the next dKV MMA may start), then
    // staged through this warp's 2 KB and stored as 64-byte row segments
    uint4* stg = sStg + (warp - 1) * 128;
    constexpr int KVW = DH / 2;                       // dKV columns of this warp
    uint32_t kvp[KVW / 2];
    auto read_kv = [&]() {
#pragma unroll
      for (int cc = 0; cc < KVW; cc += 32) {
        float v[32];
        tmem_row<32>(T_KV + lo + KVW * g + cc, v);
#pragma unroll
        for (int u = 0; u < 32; u += 2) kvp[(cc + u) / 2] = sm100::pack_bf16(v[u], v[u + 1]);
      }
    };
    auto store_kv = [&](int c) {
      const int kbase = c * kC + q * 32;
#pragma unroll
      for (int cc = 0; cc < KVW; cc += 32) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          stg[lane * 4 + (j ^ ((lane >> 1) & 3))] =
              make_uint4(kvp[(cc + 8 * j) / 2], kvp[(cc + 8 * j) / 2 + 1], kvp[(cc + 8 * j) / 2 + 2],
                         kvp[(cc + 8 * j) / 2 + 3]);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = k * 8 + (lane >> 2), sgm = lane & 3;
          if (kbase + r < a.nk)
            *reinterpret_cast<uint4*>(a.dK + (long long)b * a.sdk + (long long)(kbase + r) * a.lddk + KVW * g + cc +
                                      sgm * 8) = stg[r * 4 + (sgm ^ ((r >> 1) & 3))];
        }
        __syncwarp();
      }
    };
    // pass 2
    for (int c = 0; c < nchunk; ++c) {
      float s[32], dp[32];
      load_sd(nchunk + c, s, dp);
      const uint32_t m = vis_mask(c * kC + row);
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const bool v = (m >> u) & 1u;
        const float p = v ? __expf(fmaf(s[u], scale, -sL[c0 + u])) : 0.f;
        s[u] = p;
        dp[u] = p * (dp[u] - sD[c0 + u]) * scale;
      }
      if (c > 0) {                                      // chunk c-1's dKV / dQ' MMAs (they read Pᵀ, dSᵀ)
        sm100::mbar_wait(bar_kvd, kvdph);
        kvdph ^= 1;
        sm100::tc_fence_after();
        read_kv();
      }
      store_row(sPT, row, PT, s, 32, c0);
      store_row(sdST, row, PT, dp, 32, c0);
      signal(bar_pd);                                  // tcgen05 fence included: the dKV read is done
      if (c > 0) store_kv(c - 1);
    }
    sm100::mbar_wait(bar_kvd, kvdph);
    kvdph ^= 1;
    sm100::tc_fence_after();
    read_kv();
    store_kv(nchunk - 1);
    // dQ' rows (queries) in lanes 0..63: quarters 0 and 1
    if (q < 2) {
#pragma unroll 1
      for (int cc = (DH / 2) * g; cc < (DH / 2) * (g + 1); cc += 32) {
        float v[32];
        tmem_row<32>(T_Q + lo + cc, v);
        if (row < nq) {
          bf16* dst = a.dQ + b * a.sdq + (long long)row * a.lddq + cc;
#pragma unroll
          for (int u = 0; u < 32; u += 8)
            *reinterpret_cast<uint4*>(dst + u) =
                make_uint4(sm100::pack_bf16(v[u], v[u + 1]), sm100::pack_bf16(v[u + 2], v[u + 3]),
                           sm100::pack_bf16(v[u + 4], v[u + 5]), sm100::pack_bf16(v[u + 6], v[u + 7]));
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

// K / V tensor maps [B][nk][D] over the strided projections (false: the strides or base addresses
// miss TMA's 16-byte rules, or LONGER_ATTN_TMA=0 → thread loads).
template <int DH>
bool kv_maps(const AttnArgs& a, int pack, CUtensorMap& tK, CUtensorMap& tV) {
  if (DH < 64 || !g_knobs.attn_tma) return false;
  auto aligned = [](const void* p, long long ld, long long sb) {
    return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 8 == 0 && sb % 8 == 0;
  };
  if (!aligned(a.Kp, a.ldk, a.sk) || !aligned(a.V, a.ldv, a.sv)) return false;
  const long long cols = (long long)a.heads * DH;
  if (pack > 1)                                   // contiguous key rows of all samples (checked)
    return tma::encode_2d_bf16(&tK, a.Kp, cols, (long long)a.B * a.nk, a.ldk, 64, kC) == 0 &&
           tma::encode_2d_bf16(&tV, a.V, cols, (long long)a.B * a.nk, a.ldv, 64, kC) == 0;
  return tma::encode_3d_bf16(&tK, a.Kp, cols, a.nk, a.B, a.ldk, a.sk, 64, kC) == 0 &&
         tma::encode_3d_bf16(&tV, a.V, cols, a.nk, a.B, a.ldv, a.sv, 64, kC) == 0;
}

// samples per CTA: self-layer shapes whose queries and keys of several samples fit one tile
// (key rows contiguous across samples for the 2-D tensor map); LONGER_ATTN_PACK=0 disables.
template <int DH>
int pack_of(const AttnArgs& a) {
  if (DH > 128 || g_knobs.attn_pack == 0 || a.nq > 64 || a.nk > 64) return 1;
  if (a.sk != (long long)a.nk * a.ldk || a.sv != (long long)a.nk * a.ldv) return 1;
  const int p = std::min(kC / a.nk, 128 / a.nq);
  return std::max(1, std::min(p, a.B));
}

template <int DH, bool TMA, bool KVS = false>
int launch_fwd_t(const AttnArgs& a, const CUtensorMap& tK, const CUtensorMap& tV, int pack, cudaStream_t st) {
  const int smem = (128 * DH + std::max(128 * kC, kC * DH) + kC * DH) * 2 + 64 + 1024;
  smem_attr(xattn_fwd_kernel<DH, TMA, KVS>, 227 * 1024);
  g_launch_fence = kFenceAttnIn | kFenceAttnOut;
  launch(xattn_fwd_kernel<DH, TMA, KVS>, ((a.B + pack - 1) / pack) * a.heads, kThreads, std::max(smem, 80 * 1024), st,
         a, tK, tV, pack);
  return (int)cudaGetLastError();
}

// keys and values are the same rows (sum_kv: the absorbed cross layer)
inline bool kv_same(const AttnArgs& a) {
  return a.sum_kv && a.Kp == a.V && a.ldk == a.ldv && a.sk == a.sv;
}

template <int DH>
int launch_fwd(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tK{}, tV{};
  // the forward runs two CTAs per SM, so B·heads ≤ 296 CTAs are already one wave: packing would
  // only idle SMs (measured +10 µs per step); LONGER_ATTN_PACK=2 forces it for testing
  const int pack = g_knobs.attn_pack == 2 ? pack_of<DH>(a) : 1;
  if constexpr (DH >= 64) {
    if (kv_maps<DH>(a, pack, tK, tV)) {
      if (kv_same(a) && g_knobs.attn_kvs) return launch_fwd_t<DH, true, true>(a, tK, tV, pack, st);
      return launch_fwd_t<DH, true>(a, tK, tV, pack, st);
    }
  }
  return launch_fwd_t<DH, false>(a, tK, tV, pack, st);
}

template <int DH, bool TMA, bool SHORT, bool KVS = false>
int launch_bwd_t(const AttnArgs& a, const CUtensorMap& tK, const CUtensorMap& tV, int pack, cudaStream_t st) {
  const int QR = (DH > 128 || SHORT) ? 64 : 128, KVB = SHORT ? 2 : 1, KVT = KVS ? 1 : 2;
  const int smem = (2 * QR * DH + KVB * KVT * kC * DH + 2 * QR * kC) * 2 + 256 * 4 + 64 + 1024;
  smem_attr(xattn_bwd_kernel<DH, TMA, SHORT, KVS>, 227 * 1024);
  g_launch_fence = kFenceAttnIn | kFenceAttnOut;
  launch(xattn_bwd_kernel<DH, TMA, SHORT, KVS>, ((a.B + pack - 1) / pack) * a.heads, kThreads8,
         std::max(smem, 116 * 1024), st, a, tK, tV, pack);
  return (int)cudaGetLastError();
}

template <int DH>
int launch_bwd(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tK{}, tV{};
  const int pack = pack_of<DH>(a);
  if constexpr (DH >= 64) {
    if (kv_maps<DH>(a, pack, tK, tV)) {
      if constexpr (DH <= 128) {
        // one sample per CTA, ≤ 64 queries, several key chunks: double-buffered K / V
        if (pack == 1 && a.nq <= 64 && a.nk > kC && g_knobs.attn_short) {
          if (kv_same(a) && a.heads == 1 && g_knobs.attn_bwd_t) {
            // keys as tile rows (xattn_bwd_t_kernel)
            const int smem = (2 * kC * DH + 2 * 64 * DH + 2 * kC * 128) * 2 + 8 * 2048 + (2 * 64 + 4 * 64) * 4 +
                             2 * 64 * 4 + 16 + 16 * 8 + 1024;
            smem_attr(xattn_bwd_t_kernel<DH>, smem);
            g_launch_fence = kFenceAttnIn | kFenceAttnOut;
            launch(xattn_bwd_t_kernel<DH>, a.B, kThreads8, smem, st, a, tK);
            return (int)cudaGetLastError();
          }
          if (kv_same(a) && g_knobs.attn_kvs) return launch_bwd_t<DH, true, true, true>(a, tK, tV, pack, st);
          return launch_bwd_t<DH, true, true>(a, tK, tV, pack, st);
        }
      }
      return launch_bwd_t<DH, true, false>(a, tK, tV, pack, st);
    }
  }
  return launch_bwd_t<DH, false, false>(a, tK, tV, pack, st);
}

}  // namespace

int attn_tc_supported(const AttnArgs& a) {
  const int dh = a.D / a.heads;
  return (a.nq <= 128 && (dh == 32 || dh == 64 || dh == 128)) || (a.nq <= 64 && dh == 256);
}

int attn_tc_fwd(const AttnArgs& a, cudaStream_t st) {
  const int dh = a.D / a.heads;
  if (dh == 256) return launch_fwd<256>(a, st);
  if (dh == 128) return launch_fwd<128>(a, st);
  if (dh == 64) return launch_fwd<64>(a, st);
  if (dh == 32) return launch_fwd<32>(a, st);
  return (int)cudaErrorInvalidValue;
}

int attn_tc_bwd(const AttnArgs& a, cudaStream_t st) {
  const int dh = a.D / a.heads;
  if (dh == 256) return launch_bwd<256>(a, st);
  if (dh == 128) return launch_bwd<128>(a, st);
  if (dh == 64) return launch_bwd<64>(a, st);
  if (dh == 32) return launch_bwd<32>(a, st);
  return (int)cudaErrorInvalidValue;
}

}  // namespace longer
