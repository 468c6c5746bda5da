// frontend.cu — fused token front-end kernels (see frontend.cuh, fe_common.cuh).
//
// Restates, per token: _event_features + abs-pos (pkg/src/longrec/inputs.py:434-482), the token
// MLP (inputs.py:447-449), and merge_inner_trans (pkg/src/longrec/merge.py:83-112) with
// grouped_attention (pkg/src/longrec/tensors.py:406-444), for 128-token tiles; and the backward of
// the token MLP + featuriser (tensors.py bw closures of linear/gelu/gather_rows).
//
// CTA = warp 0 (TMEM owner + single-thread MMA issuer) + 4 worker warps (fe_fwd, two CTAs per SM)
// or 8 (fe_mlp_bwd, two per lane quadrant); thread = token row = TMEM lane.  Per stage: workers write the A tile → mbarrier → one thread issues tcgen05.mma
// (M = 128) against smem-resident weights → tcgen05.commit → workers read the fp32 accumulator
// from TMEM and apply bias / GELU / LN / group attention in registers.
#include "frontend.cuh"
#include "fe_common.cuh"

#include <algorithm>
#include <cstdlib>

namespace longer {

using namespace fe;

namespace {

// ------------------------------------------------------------------ weight packing
struct PackW {
  int n;
  struct { long long src; int in, out, trans, n_off, k_off, Kdim, dst, f16; } s[96];
};

// trans = 1: image of Wᵀ ([out][in]: element (n=j, k=i) = W[i][j]); trans = 0: image of W as
// [in][out] (element (n=i, k=j) = W[i][j]).  W is the fp32 master [in, out] row-major.
__global__ void pack_canon_kernel(const float* __restrict__ params, PackW pw, bf16* blob, ProjArgs pj) {
  pdl_trigger();
  pdl_wait();
  if (blockIdx.y == pw.n) {
    // the extra row of blocks: P[r] = table_row(r) · W_tp[cols of its table] (+ b_tp on the time
    // rows), fp32 (inputs.py:434-444 restated: the featuriser's linear map per table row, once per step)
    const int rows = pj.vocab + pj.n_actions + pj.nb, d = pj.d;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * d; e += gridDim.x * blockDim.x) {
      const int r = e / d, c = e % d;
      const float* src;
      int w, k0;
      float acc = 0.f;
      if (r < pj.vocab) { src = pj.item_tab + (long long)r * pj.d_item; w = pj.d_item; k0 = 0; }
      else if (r < pj.vocab + pj.n_actions) { src = pj.act_tab + (long long)(r - pj.vocab) * pj.d_act; w = pj.d_act; k0 = pj.d_item; }
      else {
        src = pj.time_tab + (long long)(r - pj.vocab - pj.n_actions) * pj.d_time; w = pj.d_time;
        k0 = pj.d_item + pj.d_act; acc = pj.tok_b[c];
      }
      for (int k = 0; k < w; ++k) acc = fmaf(src[k], pj.tok_w[(k0 + k) * d + c], acc);
      pj.proj[e] = acc;
    }
    return;
  }
  const auto s = pw.s[blockIdx.y];
  const int n_el = s.in * s.out;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_el; e += gridDim.x * blockDim.x) {
    const int i = e / s.out, j = e % s.out;
    const float v = params[s.src + e];
    const int idx = s.trans ? canon(s.n_off + j, s.k_off + i, s.Kdim) : canon(s.n_off + i, s.k_off + j, s.Kdim);
    if (s.f16) reinterpret_cast<__half*>(blob)[s.dst + idx] = __float2half_rn(v);
    else blob[s.dst + idx] = __float2bfloat16(v);
  }
}

// ------------------------------------------------------------------ shared worker pieces
struct TokenInfo {
  long long t;
  int b, j, n, rec;
  bool in_range, real, keep;
};

__device__ __forceinline__ TokenInfo token_info(const FrontArgs& a, long long tile, int row) {
  TokenInfo ti;
  ti.t = tile * kTile + row;
  ti.in_range = ti.t < a.T;
  ti.b = 0; ti.j = 0; ti.n = 0;
  if (ti.in_range) {
    ti.b = (int)(ti.t / a.Lp);
    ti.j = (int)(ti.t % a.Lp);
    ti.n = min(max(a.n_events[ti.b], 0), a.L);
  }
  ti.real = ti.in_range && ti.j >= a.Lp - ti.n;
  const int npg = (a.Lp - ti.n) / a.K;
  ti.keep = ti.in_range && (ti.j / a.K) >= npg;
  ti.rec = ti.real ? a.Lp - 1 - ti.j : 0;
  return ti;
}

// featuriser: concat(item, action, time-bucket embeddings), zero-padded to kFP columns, from the
// token's raw (item, action, Δt) — loaded by the caller, possibly a tile ahead
__device__ __forceinline__ void featurise_raw(const FrontArgs& a, const TokenInfo& ti, int item, int act, int dt,
                                              float* v, int* ids, bool flag) {
#pragma unroll
  for (int c = 0; c < kFP; ++c) v[c] = 0.f;
  ids[0] = ids[1] = ids[2] = 0;
  if (!ti.real) return;
  int bad = 0;
  if (item < 0 || item >= a.vocab) { bad |= 1; item = 0; }
  if (act < 0 || act >= a.n_actions) { bad |= 1; act = 0; }
  if (dt < 0) { bad |= 2; dt = 0; }
  if (bad && flag) atomicOr(a.status, bad);
  const int bucket = min(32 - __clz(dt), a.nb - 1);      // time_bucket (inputs.py:307-315)
  ids[0] = item; ids[1] = act; ids[2] = bucket;
  const int e1 = a.d_item, e2 = a.d_item + a.d_act, e3 = e2 + a.d_time;
  const float* pi = a.item_tab + item * a.d_item;
  const float* pa = a.act_tab + act * a.d_act;
  const float* pt = a.time_tab + bucket * a.d_time;
  if ((((e1 | a.d_act | a.d_time) & 3) | ((reinterpret_cast<uintptr_t>(a.item_tab) | reinterpret_cast<uintptr_t>(a.act_tab) |
                                            reinterpret_cast<uintptr_t>(a.time_tab)) & 15)) == 0) {
    // widths in multiples of 4 (16-byte rows): one float4 per 4 columns
#pragma unroll
    for (int c = 0; c < kFP; c += 4) {
      const float* p = c < e1 ? pi + c : c < e2 ? pa + (c - e1) : pt + (c - e2);
      const float4 x = c < e3 ? __ldg(reinterpret_cast<const float4*>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[c] = x.x; v[c + 1] = x.y; v[c + 2] = x.z; v[c + 3] = x.w;
    }
    return;
  }
#pragma unroll
  for (int c = 0; c < kFP; ++c) {
    const float* p = c < e1 ? a.item_tab + item * a.d_item + c
                   : c < e2 ? a.act_tab + act * a.d_act + (c - e1)
                            : a.time_tab + bucket * a.d_time + (c - e2);
    v[c] = c < e3 ? __ldg(p) : 0.f;
  }
}

// rows of FrontArgs::proj for the token's item, action and time bucket (time_bucket, inputs.py:307-315);
// out-of-range ids raise the device flag (EmbeddingLookupError / ConfigError) and read row 0
__device__ __forceinline__ void proj_rows(const FrontArgs& a, const TokenInfo& ti, int* rows) {
  int item = 0, act = 0, dt = 0;
  if (ti.real) {
    const long long src = (long long)ti.b * a.L + (ti.j - (a.Lp - a.L));
    item = a.items[src]; act = a.actions[src]; dt = a.dt[src];
    int bad = 0;
    if (item < 0 || item >= a.vocab) { bad |= 1; item = 0; }
    if (act < 0 || act >= a.n_actions) { bad |= 1; act = 0; }
    if (dt < 0) { bad |= 2; dt = 0; }
    if (bad) atomicOr(a.status, bad);
  }
  rows[0] = item;
  rows[1] = a.vocab + act;
  rows[2] = a.vocab + a.n_actions + min(32 - __clz(dt), a.nb - 1);
}

__device__ __forceinline__ void featurise(const FrontArgs& a, const TokenInfo& ti, float* v, int* ids, bool flag) {
  int item = 0, act = 0, dt = 0;
  if (ti.real) {
    const long long src = (long long)ti.b * a.L + (ti.j - (a.Lp - a.L));
    item = a.items[src]; act = a.actions[src]; dt = a.dt[src];
  }
  featurise_raw(a, ti, item, act, dt, v, ids, flag);
}

// table[id][0:width] += v[off : off+width] for every lane with id ≥ 0, summing lanes that share an id
// with warp shuffles first (one shared atomic per distinct id and column).
__device__ __forceinline__ void warp_scatter_add(float* table, int id, const float (&v)[kFP], int off, int width) {
  const int lane = threadIdx.x & 31;
  unsigned pending = __ballot_sync(0xffffffffu, id >= 0);
  while (pending) {
    const int leader = __ffs(pending) - 1;
    const int key = __shfl_sync(0xffffffffu, id, leader);
    const unsigned grp = __ballot_sync(0xffffffffu, id == key);
#pragma unroll
    for (int c = 0; c < kFP; ++c) {
      if (c >= off && c < off + width) {                  // warp-uniform
        const float s = warp_sum(id == key ? v[c] : 0.f);
        if (lane == leader) atomicAdd(table + key * width + (c - off), s);
      }
    }
    pending &= ~grp;
  }
}

__device__ __forceinline__ void load_blob(uint8_t* dst_smem, const uint8_t* src, int bytes, uint64_t* bar) {
  for (int off = 0; off < bytes; off += 32768) {
    const int n = min(32768, bytes - off);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sm100::smem_u32(dst_smem + off)), "l"(src + off), "r"(n), "r"(sm100::smem_u32(bar))
                 : "memory");
  }
}

// InnerTrans k|v scratch: row r holds [k | v] (2·DT bf16) as 16-byte chunks, chunk index XOR-ed
// with the row so that the group peers' rows (same chunk, consecutive rows) hit distinct banks.
template <int DT>
__device__ __forceinline__ void kv_store(bf16* skv, int row, const float* kv) {
  constexpr int CPR = 2 * DT / 8;
#pragma unroll
  for (int ch = 0; ch < CPR; ++ch) {
    uint4 w;
    w.x = sm100::pack_bf16(kv[8 * ch], kv[8 * ch + 1]); w.y = sm100::pack_bf16(kv[8 * ch + 2], kv[8 * ch + 3]);
    w.z = sm100::pack_bf16(kv[8 * ch + 4], kv[8 * ch + 5]); w.w = sm100::pack_bf16(kv[8 * ch + 6], kv[8 * ch + 7]);
    *reinterpret_cast<uint4*>(skv + row * 2 * DT + ((ch ^ (row % CPR)) * 8)) = w;
  }
}
// one half of the row (k: part 0, v: part 1), DT values
template <int DT>
__device__ __forceinline__ void kv_store_part(bf16* skv, int row, int part, const float* x) {
  constexpr int CPR = 2 * DT / 8;
#pragma unroll
  for (int c = 0; c < DT / 8; ++c) {
    const int ch = part * (DT / 8) + c;
    uint4 w;
    w.x = sm100::pack_bf16(x[8 * c], x[8 * c + 1]); w.y = sm100::pack_bf16(x[8 * c + 2], x[8 * c + 3]);
    w.z = sm100::pack_bf16(x[8 * c + 4], x[8 * c + 5]); w.w = sm100::pack_bf16(x[8 * c + 6], x[8 * c + 7]);
    *reinterpret_cast<uint4*>(skv + row * 2 * DT + ((ch ^ (row % CPR)) * 8)) = w;
  }
}
template <int DT>
__device__ __forceinline__ uint4 kv_raw8(const bf16* skv, int row, int col) {
  constexpr int CPR = 2 * DT / 8;
  return *reinterpret_cast<const uint4*>(skv + row * 2 * DT + (((col / 8) ^ (row % CPR)) * 8));
}

// ------------------------------------------------------------------ forward kernel
// S independent token tiles ("slots") in flight per CTA, one CTA per SM.  Slot s owns an MMA
// issuer warp (warp s, one thread), four worker warps S+4s … S+4s+3 (one per TMEM lane quadrant:
// thread = token row), TMEM columns [128s, 128s+128), an A tile and a hidden / k|v tile in shared
// memory, and a barrier pair: bar_a[s] (its 128 rows have written the next operand) and bar_d[s]
// (its MMAs are done).  Each slot alternates strictly — workers signal stage k, the issuer issues
// stage k and commits, workers wait — so a barrier never completes twice before its waiter consumed
// the phase; each issuer sleeps on its own barrier and its commits track only its own MMAs, so the
// slots never wait for each other.  While one slot's rows run GELU / LayerNorm / group attention,
// the tensor core works for another and the SIMT pipes always have 4S independent warps of work.
// The weights are loaded once per CTA and shared by all slots.
//
// Per tile (TMEM columns relative to the slot base): [feat|1]·[W_tp;b] → X [0,32);
// [x0|1]·[W1;b1] in 64-column parts → A [0,64), GELU (f16x2) → H, H·W2 (f16) accumulates h in
// [64,96); per InnerTrans layer: [LN1|1]·[Wqkv;b] → [0,96), group attention → ctx, ctx·Wo →
// [0,32), [LN2|1]·[W1;b1] parts → [0,64), GELU → H, H·W2 (f16) → [64,96).
constexpr int kSlotCols = 128;

template <int DT, int KG>
struct FwdPlan {
  static constexpr int D = DT * KG, H2 = 2 * D, nh = H2 / 64, nf = 4 * DT / 64, XK = DT + 16;
  static __host__ __device__ int stages(int IL) { return 1 + nh + IL * (3 + nf); }
};

template <int DT, int KG>
__device__ __forceinline__ void fwd_issue(int st, uint32_t t0, uint32_t wA, uint32_t wH, uint32_t wW,
                                          const BlobOff& bo) {
  using P = FwdPlan<DT, KG>;
  constexpr int XK = P::XK, nh = P::nh, nf = P::nf, H2 = P::H2;
  auto W = [&](int off, int kdim) { return Opnd{wW + off * 2, kdim, 0}; };
  auto w2mma = [&](uint32_t d, int off, int kdim, bool acc) {       // H (f16) · W2 image (f16)
    const uint32_t idesc = sm100::make_idesc_f16(128, DT, 0, 0);
    const Opnd A{wH, 64, 0}, B = W(off, kdim);
    for (int ks = 0; ks < 4; ++ks) sm100::mma_bf16(d, A.desc(ks), B.desc(ks), idesc, (acc || ks > 0) ? 1u : 0u);
  };
  if (st == 0) { mma(t0, Opnd{wA, XK, 0}, W(bo.w1, XK), XK / 16, 64, false); return; }
  st -= 1;
  if (st < nh) {
    w2mma(t0 + 64, bo.w2 + canon(0, 64 * st, H2), H2, st > 0);
    if (st + 1 < nh) mma(t0, Opnd{wA, XK, 0}, W(bo.w1 + canon(64 * (st + 1), 0, XK), XK), XK / 16, 64, false);
    return;
  }
  st -= nh;
  const int l = st / (3 + nf), r = st % (3 + nf);
  if (r == 0) { mma(t0, Opnd{wA, XK, 0}, W(bo.qkv[l], XK), XK / 16, 3 * DT, false); return; }
  if (r == 1) { mma(t0, Opnd{wA, XK, 0}, W(bo.wo[l], DT), DT / 16, DT, false); return; }
  if (r == 2) { mma(t0, Opnd{wA, XK, 0}, W(bo.w1i[l], XK), XK / 16, 64, false); return; }
  const int j = r - 3;
  w2mma(t0 + 64, bo.w2i[l] + canon(0, 64 * j, 4 * DT), 4 * DT, j > 0);
  if (j + 1 < nf) mma(t0, Opnd{wA, XK, 0}, W(bo.w1i[l] + canon(64 * (j + 1), 0, XK), XK), XK / 16, 64, false);
}

// 32 fp32 values of a row → GELU in f16 → 4 × 16-byte stores into a canonical f16 tile
__device__ __forceinline__ void gelu_store_f16(bf16* tile, int row, int kdim, int k0, const float* v) {
#pragma unroll
  for (int c = 0; c < 32; c += 8) {
    uint4 w;
    w.x = gelu2_f16(v[c], v[c + 1]); w.y = gelu2_f16(v[c + 2], v[c + 3]);
    w.z = gelu2_f16(v[c + 4], v[c + 5]); w.w = gelu2_f16(v[c + 6], v[c + 7]);
    *reinterpret_cast<uint4*>(tile + canon(row, k0 + c, kdim)) = w;
  }
}

// [· | 1 | 0 …] bias column block of an XK-wide operand row (columns DT … DT+15)
template <int DT>
__device__ __forceinline__ void store_ones_col(bf16* tile, int row) {
  constexpr int XK = DT + 16;
  *reinterpret_cast<uint4*>(tile + canon(row, DT, XK)) = make_uint4(0x3F80u, 0u, 0u, 0u);
  *reinterpret_cast<uint4*>(tile + canon(row, DT + 8, XK)) = make_uint4(0u, 0u, 0u, 0u);
}

// The warp's 32 token rows (thread = row, DT fp32 values) → dst rows [0, nvalid) (row stride DT),
// through a 32 x DT fp32 staging area (16-byte chunks XOR-swizzled by row: conflict-free both ways)
// so every store instruction writes whole 128-byte rows instead of 32 scattered 16-byte pieces.
template <int DT>
__device__ __forceinline__ void warp_store_rows_f32(float* dst, int nvalid, const float* h, float4* stg, int lane) {
  constexpr int CH = DT / 4;                          // 16-byte chunks per row
#pragma unroll
  for (int j = 0; j < CH; ++j)
    stg[lane * CH + (j ^ (lane & (CH - 1)))] = make_float4(h[4 * j], h[4 * j + 1], h[4 * j + 2], h[4 * j + 3]);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int idx = k * 32 + lane, r = idx / CH, sg = idx % CH;
    if (r < nvalid) reinterpret_cast<float4*>(dst)[r * CH + sg] = stg[r * CH + (sg ^ (r & (CH - 1)))];
  }
  __syncwarp();
}

template <int DT, int KG, int S>
__global__ void __launch_bounds__(32 * 4 * S, 1) fe_fwd_kernel(FrontArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using P = FwdPlan<DT, KG>;
  constexpr int D = P::D, nh = P::nh, nf = P::nf, XK = P::XK;
  const BlobOff bo = blob_offsets(DT, D, a.inner_layers);
  bf16* sW = reinterpret_cast<bf16*>(smem_raw);
  bf16* sA0 = sW + ((bo.fwd_total + 63) & ~63);               // S x [128 x XK] bf16 (feat: 128 x 32)
  bf16* sH0 = sA0 + S * kTile * XK;                           // S x [128 x 64] f16 hidden / bf16 k|v
  float* s_par = reinterpret_cast<float*>(sH0 + S * kTile * 64);   // [IL][ln1_g, ln1_b, b_o, ln2_g, ln2_b, b2]
  float* s_b2 = s_par + a.inner_layers * 6 * DT;              // token-MLP output bias [DT]
  float* s_kn = s_b2 + DT;                                    // cross LN1 [gain | bias] (2D)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_kn + (a.kn_global ? 0 : 2 * D));
  uint64_t* bar_w = bars;
  uint64_t* bar_a = bars + 1;                                 // [S]
  uint64_t* bar_d = bars + 1 + S;                             // [S]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 1 + 2 * S);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_w, 1);
    for (int s = 0; s < S; ++s) {
      sm100::mbar_init(&bar_a[s], 128);
      sm100::mbar_init(&bar_d[s], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  for (int i = threadIdx.x; i < a.inner_layers * 6 * DT; i += blockDim.x) {
    const int l = i / (6 * DT), v = (i / DT) % 6, c = i % DT;
    const float* src = v == 0 ? a.inner_ln[l][0] : v == 1 ? a.inner_ln[l][1] : v == 2 ? a.inner_bias[l][3]
                     : v == 3 ? a.inner_ln[l][2] : v == 4 ? a.inner_ln[l][3] : a.inner_bias[l][5];
    s_par[i] = src[c];
  }
  for (int i = threadIdx.x; i < DT; i += blockDim.x) s_b2[i] = a.seq_b2[i];
  if (a.kn && !a.kn_global)
    for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) s_kn[i] = i < D ? a.kn_g[i] : a.kn_b[i - D];
  __syncthreads();
  const long long ntiles = (a.T + kTile - 1) / kTile;
  const long long stride = (long long)gridDim.x * S;

  // The MMA issuer of slot s is lane 0 of the slot's first worker warp: right after its own arrival
  // it waits for the slot's other 127 rows, issues the stage and commits (a commit tracks only this
  // thread's MMAs: slots never wait for each other).  No separate issuer warps: 16 warps, so ptxas
  // budgets 128 registers per thread instead of 96 (it sizes the budget for the CTA's warps).
  if (threadIdx.x == 0) {
    sm100::mbar_arrive_expect_tx(bar_w, bo.fwd_total * 2);
    load_blob(reinterpret_cast<uint8_t*>(sW), reinterpret_cast<const uint8_t*>(a.wblob), bo.fwd_total * 2, bar_w);
  }
  {
    // ---------------- workers: slot s, one token row per thread
    const int s = warp >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t trow = tmem + s * kSlotCols + ((uint32_t)(q * 32) << 16);
    bf16* sA = sA0 + s * kTile * XK;
    bf16* sH = sH0 + s * kTile * 64;
    bf16* sKV = sH;                                  // 128 x 2DT bf16, 16-byte chunks XOR-swizzled
    const float scale_in = rsqrtf((float)DT);
    uint32_t pd = 0;
    const bool issuer = q == 0 && lane == 0;
    const int NS = P::stages(a.inner_layers);
    const uint32_t wW = sm100::smem_u32(sW), wA = sm100::smem_u32(sA0 + s * kTile * XK);
    const uint32_t wH = sm100::smem_u32(sH0 + s * kTile * 64), tslot = tmem + s * kSlotCols;
    uint32_t pa = 0;
    int st_i = 0;
    bool w_ready = false;
    auto signal = [&]() {
      sm100::fence_async_smem();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&bar_a[s]);
      if (issuer) {
        if (!w_ready) { sm100::mbar_wait(bar_w, 0); w_ready = true; }
        sm100::mbar_wait(&bar_a[s], pa);
        pa ^= 1;
        sm100::tc_fence_after();
        fwd_issue<DT, KG>(st_i, tslot, wA, wH, wW, bo);
        sm100::mma_commit(&bar_d[s]);
        if (++st_i == NS) st_i = 0;
      }
    };
    auto wait_d = [&]() { sm100::mbar_wait(&bar_d[s], pd); pd ^= 1; sm100::tc_fence_after(); };
    for (long long tile = (long long)blockIdx.x * S + s; tile < ntiles; tile += stride) {
      const TokenInfo ti = token_info(a, tile, row);
      if (ti.in_range && ti.j == 0 && a.npg) a.npg[ti.b] = (a.Lp - ti.n) / a.K;
      if (ti.in_range && a.real_out) {
        a.real_out[ti.t] = ti.real ? 1.f : 0.f;
        a.keep_out[ti.t] = ti.keep ? 1.f : 0.f;
      }
      float h[DT];
      {
        // x0 = P[item] + P[action] + P[bucket] + abs_pos[recency]  (the featuriser's tok_proj
        // applied per table row: FrontArgs::proj).  The warp gathers its 32 rows cooperatively —
        // DT / 4 lanes per row, one float4 each, so one load instruction covers whole 128-byte
        // rows of 32 / (DT / 4) tokens instead of 32 scattered 16-byte pieces — and writes x0
        // straight into its rows of the canonical A tile.
        int pr[3];
        proj_rows(a, ti, pr);
        constexpr int LPR = DT / 4, RPS = 32 / LPR;      // lanes per row, rows per step
        const int sub = lane % LPR, rsel = lane / LPR;
#pragma unroll
        for (int st = 0; st < 32 / RPS; ++st) {
          const int r = st * RPS + rsel;
          const int i0 = __shfl_sync(0xffffffffu, pr[0], r), i1 = __shfl_sync(0xffffffffu, pr[1], r);
          const int i2 = __shfl_sync(0xffffffffu, pr[2], r), rc = __shfl_sync(0xffffffffu, ti.rec, r);
          const bool re = __shfl_sync(0xffffffffu, (int)ti.real, r) != 0;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (re) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(a.pos_tab + (long long)rc * DT) + sub);
            const float4 y0 = __ldg(reinterpret_cast<const float4*>(a.proj + (long long)i0 * DT) + sub);
            const float4 y1 = __ldg(reinterpret_cast<const float4*>(a.proj + (long long)i1 * DT) + sub);
            const float4 y2 = __ldg(reinterpret_cast<const float4*>(a.proj + (long long)i2 * DT) + sub);
            v = make_float4((y0.x + y1.x) + (y2.x + x.x), (y0.y + y1.y) + (y2.y + x.y), (y0.z + y1.z) + (y2.z + x.z),
                            (y0.w + y1.w) + (y2.w + x.w));
          }
          *reinterpret_cast<uint2*>(sA + canon(q * 32 + r, 4 * sub, XK)) =
              make_uint2(sm100::pack_bf16(v.x, v.y), sm100::pack_bf16(v.z, v.w));
        }
        store_ones_col<DT>(sA, row);
      }
      signal();
      // token MLP: GELU([x0 | 1]·[W1 ; b1]) in 64-column parts (f16) · W2 accumulates in TMEM
      for (int hj = 0; hj < nh; ++hj) {
        wait_d();
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 32) {
          float hv[32];
          tmem_row<32>(trow + c0, hv);
          gelu_store_f16(sH, row, 64, c0, hv);
        }
        signal();
      }
      wait_d();
      tmem_row<DT>(trow + 64, h);
#pragma unroll
      for (int c = 0; c < DT; ++c) h[c] = ti.real ? h[c] + s_b2[c] : 0.f;
      // rows staged through this warp's quarter of the slot's hidden tile (its W2 MMAs are done;
      // the next writer is the k|v scratch after the QKV wait)
      float4* stg = reinterpret_cast<float4*>(sH) + q * (32 * DT / 4);
      const long long t0 = tile * kTile + q * 32;
      const int nvalid = a.T - t0 < 32 ? (int)(a.T - t0) : 32;
      if (a.h_out) warp_store_rows_f32<DT>(a.h_out + t0 * DT, nvalid, h, stg, lane);
      // the residual stream h is parked in the slot's TMEM columns [96, 128) while the attention
      // and FFN stages run (registers: 4S warps share the SM)
      const uint32_t tres = trow + 96;
      for (int l = 0; l < a.inner_layers; ++l) {
        const float* par = s_par + l * 6 * DT;
        {
          float xn[DT], inv;
          ln_row_s<DT>(h, par, par + DT, xn, inv);
          store_row(sA, row, XK, xn, DT);
          store_ones_col<DT>(sA, row);
        }
        tmem_row_st<DT>(tres, h);
        signal();
        wait_d();
        float ctx[DT];
        {
          float kv[DT];                              // q, k, v already carry their biases
          tmem_row<DT>(trow + DT, kv);
          kv_store_part<DT>(sKV, row, 0, kv);
          tmem_row<DT>(trow + 2 * DT, kv);
          kv_store_part<DT>(sKV, row, 1, kv);
        }
        __syncwarp();
        {
          // scores and context with fp32 += bf16·bf16 FMAs (q rounded to bf16 like k and v; the
          // probabilities rounded to bf16 for the context)
          uint32_t qp[DT / 2];
          {
            float qv[DT];
            tmem_row<DT>(trow, qv);
#pragma unroll
            for (int c = 0; c < DT; c += 2) qp[c / 2] = sm100::pack_bf16(qv[c], qv[c + 1]);
          }
          const int g0 = row - row % KG;
          float sc[KG];
          float mx = -INFINITY;
#pragma unroll
          for (int jj = 0; jj < KG; ++jj) {
            float acc = 0.f;
#pragma unroll
            for (int c = 0; c < DT; c += 8) {
              const uint4 w = kv_raw8<DT>(sKV, g0 + jj, c);
              acc = sm100::dot2_bf16(qp[c / 2], w.x, acc);
              acc = sm100::dot2_bf16(qp[c / 2 + 1], w.y, acc);
              acc = sm100::dot2_bf16(qp[c / 2 + 2], w.z, acc);
              acc = sm100::dot2_bf16(qp[c / 2 + 3], w.w, acc);
            }
            sc[jj] = acc * scale_in;
            mx = fmaxf(mx, sc[jj]);
          }
          float tot = 0.f;
#pragma unroll
          for (int jj = 0; jj < KG; ++jj) { sc[jj] = __expf(sc[jj] - mx); tot += sc[jj]; }
          const float rinv = 1.f / tot;
#pragma unroll
          for (int c = 0; c < DT; ++c) ctx[c] = 0.f;
#pragma unroll
          for (int jj = 0; jj < KG; ++jj) {
            const uint32_t pj = sm100::bf16_scalar(sc[jj] * rinv);
#pragma unroll
            for (int c = 0; c < DT; c += 8) {
              const uint4 w = kv_raw8<DT>(sKV, g0 + jj, DT + c);
              sm100::axpy2_bf16(pj, w.x, ctx[c], ctx[c + 1]);
              sm100::axpy2_bf16(pj, w.y, ctx[c + 2], ctx[c + 3]);
              sm100::axpy2_bf16(pj, w.z, ctx[c + 4], ctx[c + 5]);
              sm100::axpy2_bf16(pj, w.w, ctx[c + 6], ctx[c + 7]);
            }
          }
        }
        __syncwarp();
        store_row(sA, row, XK, ctx, DT);
        store_ones_col<DT>(sA, row);                   // Woᵀ has K = DT: the ones column is unread
        signal();
        wait_d();
        {
          float o[DT];
          tmem_row<DT>(trow, o);
          tmem_row<DT>(tres, h);
#pragma unroll
          for (int c = 0; c < DT; ++c) h[c] += o[c] + par[2 * DT + c];      // x1
          float xn[DT], inv;
          ln_row_s<DT>(h, par + 3 * DT, par + 4 * DT, xn, inv);
          store_row(sA, row, XK, xn, DT);
          store_ones_col<DT>(sA, row);
          tmem_row_st<DT>(tres, h);
        }
        signal();
        for (int fj = 0; fj < nf; ++fj) {
          wait_d();
#pragma unroll
          for (int c0 = 0; c0 < 64; c0 += 32) {
            float hv[32];
            tmem_row<32>(trow + c0, hv);
            gelu_store_f16(sH, row, 64, c0, hv);
          }
          signal();
        }
        wait_d();
        {
          float o[DT];
          tmem_row<DT>(trow + 64, o);
          tmem_row<DT>(tres, h);
#pragma unroll
          for (int c = 0; c < DT; ++c) h[c] += o[c] + par[5 * DT + c];      // x2
        }
      }
      if (a.inner_layers > 0 && !ti.keep) {
#pragma unroll
        for (int c = 0; c < DT; ++c) h[c] = 0.f;
      }
      warp_store_rows_f32<DT>(a.merged + t0 * DT, nvalid, h, stg, lane);   // sH free: W2 MMAs done
      if (a.kn) {
        // cross LN1 of the merged row = the KG consecutive tokens of this group (adjacent lanes)
        float s1 = 0.f;
#pragma unroll
        for (int c = 0; c < DT; ++c) s1 += h[c];
#pragma unroll
        for (int o2 = 1; o2 < KG; o2 <<= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, o2);
        const float mu = s1 * (1.f / D);
        float s2 = 0.f;
#pragma unroll
        for (int c = 0; c < DT; ++c) { const float t = h[c] - mu; s2 += t * t; }
#pragma unroll
        for (int o2 = 1; o2 < KG; o2 <<= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o2);
        const float inv = rsqrtf(s2 * (1.f / D) + kLnEps);
        if (ti.in_range) {
          const int part = ti.j % KG;
          const long long krow = (long long)ti.b * a.v + ti.j / KG;
          bf16* dst = a.kn + krow * D + part * DT;
          const float* gk = (a.kn_global ? a.kn_g : s_kn) + part * DT;
          const float* bk = (a.kn_global ? a.kn_b : s_kn + D) + part * DT;
#pragma unroll
          for (int c = 0; c < DT; c += 8) {
            const float4 g0 = *reinterpret_cast<const float4*>(gk + c), g1 = *reinterpret_cast<const float4*>(gk + c + 4);
            const float4 b0 = *reinterpret_cast<const float4*>(bk + c), b1 = *reinterpret_cast<const float4*>(bk + c + 4);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            float y[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) y[u] = fmaf((h[c + u] - mu) * inv, gg[u], bb[u]);
            uint4 w;
            w.x = sm100::pack_bf16(y[0], y[1]); w.y = sm100::pack_bf16(y[2], y[3]);
            w.z = sm100::pack_bf16(y[4], y[5]); w.w = sm100::pack_bf16(y[6], y[7]);
            *reinterpret_cast<uint4*>(dst + c) = w;
          }
          if (part == 0) { a.kn_mean[krow] = mu; a.kn_rstd[krow] = inv; }
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ token-MLP + featuriser backward
// Per tile: recompute feat, x0 and the hidden a1 (one 128-column half at a time), then
//   da1 = (dh·W2ᵀ) ⊙ GELU'(a1),   dx0 = da1·W1ᵀ,   dfeat = dx0·W_tpᵀ
// and accumulate, in TMEM for the whole kernel:
//   dW2 += g1ᵀ·dh,   [dW1ᵀ | db1] += da1ᵀ·[x0 | 1],
//   [dW_tpᵀ | db_tp ; · | db2] += [dx0 | dh]ᵀ·[feat | 1]       (bias sums from the ones column)
//   Y += onehot([bucket | action])ᵀ·dx0                        (time / action table grads = Y·W_tpᵀ)
// Tiles are column blocks of one sample (token position fixed per thread for the whole kernel), so
// the abs-pos rows are loaded once and their gradient accumulates in shared memory.
template <int DT>
__global__ void __launch_bounds__(kThreads8, 1) fe_mlp_bwd_kernel(FrontArgs a) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int Dm = DT * a.K;
  const int H2 = 2 * Dm;
  // this launch's hidden units [h0, h0 + HP) (all of them unless the MLP runs in passes)
  const int h0 = a.mlp_hn ? a.mlp_h0 : 0, HP = a.mlp_hn ? a.mlp_hn : H2;
  const bool last = a.mlp_last != 0;
  const int nh = HP / 128;
  const int XK = DT + 16;                  // x0 tile row: [x0 | 1 | 0…] for the db1 column
  const BlobOff bo = blob_offsets(DT, Dm, a.inner_layers);
  // smem carve-up (the weight images of this pass's hidden slice)
  bf16* sW = reinterpret_cast<bf16*>(smem_raw);                    // tp, w1 (fwd) + tp_n, w1_n, w2_n
  const int n_tp = DT * kFP, n_w1 = HP * DT, n_w1f = HP * XK;
  bf16* w_tp = sW;
  bf16* w_w1 = w_tp + n_tp;                    // [W1ᵀ | b1] image, K = XK
  bf16* w_tp_n = w_w1 + n_w1f;
  bf16* w_w1_n = w_tp_n + n_tp;
  bf16* w_w2_n = w_w1_n + n_w1;
  bf16* sFeat = w_w2_n + n_w1;                 // 128 x 32   [feat | 1]
  bf16* sX0 = sFeat + kTile * kFP;             // 128 x XK   [x0 | 1]
  bf16* sDH = sX0 + kTile * XK;                // 128 x DT
  bf16* sG = sDH + kTile * DT;                 // 128 x 128
  bf16* sDA = sG + kTile * 128;                // 128 x 128
  bf16* sDX0 = sDA + kTile * 128;              // 128 x 64   [dx0 | dh]
  bf16* sOH = sDX0 + kTile * 64;               // 128 x 64   [onehot(bucket) | onehot(action)]
  float* s_pos = reinterpret_cast<float*>(sOH + kTile * 64);        // 128 x (DT+1)
  float* s_gpos = s_pos + kTile * (DT + 1);                         // 128 x (DT+1)
  float* s_item = s_gpos + kTile * (DT + 1);
  const int n_item = a.vocab * a.d_item;
  const bool item_smem = a.item_smem && n_item <= 16384;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_item + (item_smem ? n_item : 0) + 2);
  bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bars) + 7) & ~uintptr_t(7));
  uint64_t* bar_w = bars;
  uint64_t* bar_a = bars + 1;
  uint64_t* bar_d = bars + 2;
  uint64_t* bar_g = bars + 3;    // the dW_tp / one-hot MMAs done (they read sFeat / sOH / sDX0)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  // column-block tiling: this CTA owns token positions [cb*128, cb*128+128) of samples b0, b0+r, …
  // (tiles t = 0, 1, … of its sequence); split mode: tiles [t0, t1) of the column-block-major
  // order (column block t / B, sample t % B) — the column block changes inside the range
  const int tps = (a.Lp + kTile - 1) / kTile;
  const bool split = a.mlp_split;
  const int r = split ? 1 : gridDim.x / tps;
  const int b0 = split ? 0 : blockIdx.x / tps;
  int t0 = 0, t1 = 0;
  if (split) {
    const long long W = (long long)tps * a.B;
    t0 = (int)(W * blockIdx.x / gridDim.x);
    t1 = (int)(W * (blockIdx.x + 1) / gridDim.x);
  } else if (b0 < a.B) {
    t1 = (a.B - b0 + r - 1) / r;
  }
  auto tile_cb = [&](int t) { return split ? t / a.B : (int)(blockIdx.x % tps); };
  auto tile_b = [&](int t) { return split ? t % a.B : b0 + t * r; };
  const int cb = t0 < t1 ? tile_cb(t0) : 0;                   // column block of the first tile
  const int cb_last = t0 < t1 ? tile_cb(t1 - 1) : 0;
  for (int i = threadIdx.x; i < (item_smem ? n_item : 0); i += blockDim.x) s_item[i] = 0.f;
  for (int i = threadIdx.x; i < kTile * DT; i += blockDim.x) {
    const int rr = i / DT, c = i % DT;
    const int rec = a.Lp - 1 - (cb * kTile + rr);
    s_pos[rr * (DT + 1) + c] = (rec >= 0 && rec < a.L) ? a.pos_tab[(long long)rec * DT + c] : 0.f;
    s_gpos[rr * (DT + 1) + c] = 0.f;
  }
  // the one-hot tile stays zero apart from each row's two ones (rewritten per tile)
  for (int i = threadIdx.x; i < kTile * 64 / 8; i += blockDim.x) reinterpret_cast<uint4*>(sOH)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_w, 1);
    sm100::mbar_init(bar_a, 32 * 2 * kWorkers);
    sm100::mbar_init(bar_d, 1);
    sm100::mbar_init(bar_g, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // TMEM columns
  const uint32_t T_DW2 = tmem;                         // nh x DT
  const uint32_t T_DW1 = tmem + nh * DT;               // nh x XK
  const uint32_t T_DWTP = tmem + 160;                  // 32: [dWtpᵀ | db_tp] rows 0..DT, db2 rows DT..2DT (col 31)
  const uint32_t T_Y = tmem + 192;                     // 32: onehotᵀ·dx0
  const uint32_t T_X = tmem + 224;                     // 32: x0 acc → dx0 acc → dfeat
  const uint32_t T_A1 = tmem + 256;                    // 128
  const uint32_t T_G1 = tmem + 384;                    // 128

  if (warp == 0) {
    if (lane == 0) {
      sm100::mbar_arrive_expect_tx(bar_w, (2 * n_tp + n_w1f + 2 * n_w1) * 2);
      auto copy = [&](bf16* dst, long long src_off, int elems) {
        load_blob(reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(a.wblob + src_off), elems * 2, bar_w);
      };
      copy(w_tp, bo.tp, n_tp);
      copy(w_w1, bo.w1 + (long long)h0 * XK, n_w1f);                 // rows h0.. of [W1ᵀ | b1]
      copy(w_tp_n, bo.tp_n, n_tp);
      // W1 (backward image, K = 2D): columns [h0, h0 + HP) of each 8-row group are contiguous
      for (int g8 = 0; g8 < DT / 8; ++g8) copy(w_w1_n + g8 * HP * 8, bo.w1_n + (long long)g8 * H2 * 8 + h0 * 8, HP * 8);
      copy(w_w2_n, bo.w2_n + (long long)h0 * DT, n_w1);              // rows h0.. of W2 (K = d)
      sm100::mbar_wait(bar_w, 0);
      const uint32_t aW1 = sm100::smem_u32(w_w1), aTP = sm100::smem_u32(w_tp), aTPn = sm100::smem_u32(w_tp_n);
      const uint32_t aW1n = sm100::smem_u32(w_w1_n), aW2n = sm100::smem_u32(w_w2_n);
      const uint32_t aFeat = sm100::smem_u32(sFeat), aX0 = sm100::smem_u32(sX0), aDH = sm100::smem_u32(sDH);
      const uint32_t aG = sm100::smem_u32(sG), aDA = sm100::smem_u32(sDA), aDX0 = sm100::smem_u32(sDX0);
      const uint32_t aOH = sm100::smem_u32(sOH);
      uint32_t pa = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      bool first = true;
      for (int t = t0; t < t1; ++t) {
        wait_a();                                                        // feat, dh, onehot
        mma(T_X, Opnd{aFeat, kFP, 0}, Opnd{aTP, kFP, 0}, kFP / 16, DT, false);
        sm100::mma_commit(bar_d);
        wait_a();                                                        // x0
        mma(T_A1, Opnd{aX0, XK, 0}, Opnd{aW1, XK, 0}, XK / 16, 128, false);
        mma(T_G1, Opnd{aDH, DT, 0}, Opnd{aW2n, DT, 0}, DT / 16, 128, false);
        sm100::mma_commit(bar_d);
        for (int j = 0; j < nh; ++j) {
          wait_a();                                                      // g1, da1 of half j
          if (j + 1 < nh) {
            // the next half's a1 / g1 first (the workers wait for them), then this half's weight
            // gradients and dx0 part behind the second barrier (the workers wait for it only before
            // they overwrite sG / sDA)
            mma(T_A1, Opnd{aX0, XK, 0}, Opnd{aW1 + canon(128 * (j + 1), 0, XK) * 2, XK, 0}, XK / 16, 128, false);
            mma(T_G1, Opnd{aDH, DT, 0}, Opnd{aW2n + canon(128 * (j + 1), 0, DT) * 2, DT, 0}, DT / 16, 128, false);
            sm100::mma_commit(bar_d);
            mma(T_DW2 + j * DT, Opnd{aG, 128, 1}, Opnd{aDH, DT, 1}, kTile / 16, DT, !first);
            mma(T_DW1 + j * XK, Opnd{aDA, 128, 1}, Opnd{aX0, XK, 1}, kTile / 16, XK, !first);
            mma(T_X, Opnd{aDA, 128, 0}, Opnd{aW1n + canon(0, 128 * j, HP) * 2, HP, 0}, 8, DT, j > 0);
            sm100::mma_commit(bar_g);
          } else {
            // last half: the workers only wait for dx0 (T_X); the weight-gradient MMAs run on
            // behind that commit (sG / sDA / sDH / sX0 are next rewritten after the tile's final
            // commit, which covers them)
            mma(T_X, Opnd{aDA, 128, 0}, Opnd{aW1n + canon(0, 128 * j, HP) * 2, HP, 0}, 8, DT, j > 0);
            if (!last) {      // no later commit in this tile: this one covers the dW MMAs too
              mma(T_DW2 + j * DT, Opnd{aG, 128, 1}, Opnd{aDH, DT, 1}, kTile / 16, DT, !first);
              mma(T_DW1 + j * XK, Opnd{aDA, 128, 1}, Opnd{aX0, XK, 1}, kTile / 16, XK, !first);
            }
            sm100::mma_commit(bar_d);
            if (last) {
              mma(T_DW2 + j * DT, Opnd{aG, 128, 1}, Opnd{aDH, DT, 1}, kTile / 16, DT, !first);
              mma(T_DW1 + j * XK, Opnd{aDA, 128, 1}, Opnd{aX0, XK, 1}, kTile / 16, XK, !first);
            }
          }
        }
        if (last) {
          wait_a();                                                      // dx0 in sDX0
          mma(T_X, Opnd{aDX0, 64, 0}, Opnd{aTPn, DT, 0}, DT / 16, kFP, false);     // dfeat first
          sm100::mma_commit(bar_d);
          mma(T_DWTP, Opnd{aDX0, 64, 1}, Opnd{aFeat, kFP, 1}, kTile / 16, kFP, !first);
          mma(T_Y, Opnd{aOH, 64, 1}, Opnd{aDX0, 64, 1}, kTile / 16, DT, !first);
          sm100::mma_commit(bar_g);                                      // sFeat / sOH / sDX0 free
        }
        first = false;
      }
    }
  } else {
    // 8 worker warps: two per TMEM lane quarter.  Group 0 (warps 1-4) and group 1 (warps 5-8) see the
    // same 32 token rows; the wide GELU/GELU' stage is split by columns, the row-wise stages by task.
    const int q = warp & 3;
    const int grp = (warp - 1) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // s_pos / s_gpos entries (row, c0..c0+XH) are read and written only by this thread: a change of
    // column block flushes / reloads them here without a CTA barrier
    int cur_cb = cb;
    uint32_t pd = 0, pg = 0;
    auto signal = [&]() { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar_a); };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    auto wait_g = [&]() { sm100::mbar_wait(bar_g, pg); pg ^= 1; sm100::tc_fence_after(); };
    // the next sample's raw inputs (n_events, ids, dh) are loaded a tile ahead, right after the
    // current tile's first stage, so their latency overlaps the MMA round trips
    int n_pf = 0, item_pf = 0, act_pf = 0, dt_pf = 0;
    uint4 dh_pf[DT / 8];                               // packed bf16 (the MMA operand type)
    auto prefetch = [&](int tt) {
      const int bb = tile_b(tt), j = tile_cb(tt) * kTile + row;
      n_pf = a.n_events[bb];
      if (j >= a.Lp) return;
      const long long src = (long long)bb * a.L + max(j - (a.Lp - a.L), 0);
      item_pf = a.items[src];
      if (grp == 0) {
        act_pf = a.actions[src];
        dt_pf = a.dt[src];
      } else {
        if (a.dh_bf) {
          const uint4* srcb = reinterpret_cast<const uint4*>(a.dh_bf + ((long long)bb * a.Lp + j) * DT);
#pragma unroll
          for (int c = 0; c < DT / 8; ++c) dh_pf[c] = srcb[c];
        } else {
          const float4* srcd = reinterpret_cast<const float4*>(a.dh + ((long long)bb * a.Lp + j) * DT);
#pragma unroll
          for (int c = 0; c < DT / 8; ++c) {
            const float4 f0 = srcd[2 * c], f1 = srcd[2 * c + 1];
            dh_pf[c] = make_uint4(sm100::pack_bf16(f0.x, f0.y), sm100::pack_bf16(f0.z, f0.w),
                                  sm100::pack_bf16(f1.x, f1.y), sm100::pack_bf16(f1.z, f1.w));
          }
        }
      }
    };
    if (t0 < t1) prefetch(t0);
    int my_tiles = 0;
    int oh_b = -1, oh_a = -1;                          // this row's one-hot columns in sOH
    // stage A of a tile: its feature / one-hot / dh rows into shared memory (from the prefetched
    // raw inputs), then the signal for its feat·W_tp MMA.  It runs for tile b+r right after tile
    // b's last MMAs (which read those tiles) completed, before tile b's item-gradient CAS loop,
    // so that loop overlaps the next tile's first MMA round trip.
    TokenInfo ti;
    int cas_item = 0;
    auto stage_a = [&](int tt) {
      const int bb = tile_b(tt), j = tile_cb(tt) * kTile + row;
      const bool col_ok = j < a.Lp;
      ti.b = bb; ti.j = j;
      ti.in_range = col_ok;
      ti.t = (long long)bb * a.Lp + j;
      ti.n = min(max(n_pf, 0), a.L);
      ti.real = col_ok && j >= a.Lp - ti.n;
      ti.keep = col_ok && (j / a.K) >= (a.Lp - ti.n) / a.K;
      ti.rec = ti.real ? a.Lp - 1 - j : 0;
      int ids[3] = {0, 0, 0};
      if (grp == 0) {
        float v[kFP];
        featurise_raw(a, ti, item_pf, act_pf, dt_pf, v, ids, false);
        v[kFP - 1] = 1.f;                                              // bias column
        store_row(sFeat, row, kFP, v, kFP);
        // [onehot(bucket) | onehot(action)]: clear the previous tile's two ones, set this tile's
        const bf16 one = __float2bfloat16(1.f), zero = __float2bfloat16(0.f);
        if (oh_b >= 0) { sOH[canon(row, oh_b, 64)] = zero; sOH[canon(row, oh_a, 64)] = zero; }
        oh_b = ti.real ? ids[2] : -1;
        oh_a = ti.real ? 32 + ids[1] : -1;
        if (oh_b >= 0) { sOH[canon(row, oh_b, 64)] = one; sOH[canon(row, oh_a, 64)] = one; }
      } else {
#pragma unroll
        for (int c = 0; c < DT / 8; ++c) {
          const uint4 v = ti.real ? dh_pf[c] : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(sDH + canon(row, 8 * c, DT)) = v;
          *reinterpret_cast<uint4*>(sDX0 + canon(row, 32 + 8 * c, 64)) = v;   // [· | dh] for the db2 row sums
        }
        if (ti.real) ids[0] = (item_pf < 0 || item_pf >= a.vocab) ? 0 : item_pf;   // for the dfeat split
      }
      cas_item = ids[0];
      signal();
      // passes after the first read this tile's partial dx0 at its end: pull the rows into L2 now
      if (h0 > 0 && col_ok) sm100::prefetch_l2(a.dx0_part + ((long long)bb * a.Lp + j) * DT + grp * (DT / 2));
    };
    if (t0 < t1) {
      stage_a(t0);
      if (t0 + 1 < t1) prefetch(t0 + 1);
    }
    for (int t = t0; t < t1; ++t, ++my_tiles) {
      const int b = tile_b(t), tcb = tile_cb(t), j = tcb * kTile + row;
      const bool col_ok = j < a.Lp;
      wait_d();
      // x0 recompute; with DT = 32 the two groups take 16 columns each
      constexpr int XH = (DT % 32 == 0) ? DT / 2 : DT;
      if (XH < DT || grp == 0) {
        const int c0 = XH < DT ? grp * XH : 0;
        if (tcb != cur_cb) {                                           // split mode: next column block
          const int rec0 = a.Lp - 1 - (cur_cb * kTile + row), rec1 = a.Lp - 1 - j;
          for (int c = 0; c < XH; ++c) {
            float& g = s_gpos[row * (DT + 1) + c0 + c];
            if (rec0 >= 0 && rec0 < a.L && g != 0.f) atomicAdd(a.g_pos + (long long)rec0 * DT + c0 + c, g);
            g = 0.f;
            s_pos[row * (DT + 1) + c0 + c] = (rec1 >= 0 && rec1 < a.L) ? a.pos_tab[(long long)rec1 * DT + c0 + c] : 0.f;
          }
          cur_cb = tcb;
        }
        float x[XH], acc[XH];
        tmem_row<XH>(T_X + lane_off + c0, acc);
#pragma unroll
        for (int c = 0; c < XH; ++c) x[c] = ti.real ? acc[c] + s_pos[row * (DT + 1) + c0 + c] : 0.f;
        store_row(sX0, row, XK, x, XH, c0);
      }
      if (grp == 1 || XH == DT) {
        if (grp == (XH < DT ? 1 : 0)) {
          float pad[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) pad[c] = c == 0 ? 1.f : 0.f;    // [· | 1 | 0…] bias column
          store_row(sX0, row, XK, pad, 16, DT);
        }
      }
      signal();
      for (int hj = 0; hj < nh; ++hj) {
        wait_d();
#pragma unroll 1
        for (int c0 = 64 * grp; c0 < 64 * grp + 64; c0 += 32) {
          float av[32], gv[32];
          tmem_row2<32>(T_A1 + lane_off + c0, av, T_G1 + lane_off + c0, gv);
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            float gd;                                               // b1 added by the MMA
            av[u] = gelu_and_grad(av[u], gd);
            gv[u] *= gd;
          }
          if (hj > 0 && c0 == 64 * grp) wait_g();                   // previous half's dW MMAs read sG / sDA
          store_row(sG, row, 128, av, 32, c0);
          store_row(sDA, row, 128, gv, 32, c0);
        }
        signal();
      }
      wait_d();
      if (XH < DT || grp == 0) {
        const int c0 = XH < DT ? grp * XH : 0;
        float dx0[XH];
        tmem_row<XH>(T_X + lane_off + c0, dx0);
        float* part = a.dx0_part ? a.dx0_part + ((long long)b * a.Lp + j) * DT + c0 : nullptr;
        if (h0 > 0 && col_ok) {                                        // earlier passes' hidden units
#pragma unroll
          for (int c = 0; c < XH; c += 4) {
            const float4 pv = *reinterpret_cast<const float4*>(part + c);
            dx0[c] += pv.x; dx0[c + 1] += pv.y; dx0[c + 2] += pv.z; dx0[c + 3] += pv.w;
          }
        }
        if (!last) {                                                   // hand the partial on
          if (col_ok) {
#pragma unroll
            for (int c = 0; c < XH; c += 4)
              *reinterpret_cast<float4*>(part + c) = make_float4(dx0[c], dx0[c + 1], dx0[c + 2], dx0[c + 3]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < XH; ++c) {
            dx0[c] = ti.real ? dx0[c] : 0.f;
            s_gpos[row * (DT + 1) + c0 + c] += dx0[c];                 // abs-pos row of this position
          }
          store_row(sDX0, row, 64, dx0, XH, c0);
        }
      }
      if (!last) {                                                     // no featuriser part in this pass
        if (t + 1 < t1) {
          stage_a(t + 1);
          if (t + 2 < t1) prefetch(t + 2);
        }
        continue;
      }
      signal();
      wait_d();
      {                                                                // item rows: dfeat[:d_item]
        float df[kFP];
        tmem_row<kFP>(T_X + lane_off, df);
        wait_g();                                                      // dW_tp / Y MMAs done
        const bool cas_real = ti.real;
        const int cas_tile_item = cas_item;
        if (t + 1 < t1) {
          stage_a(t + 1);
          if (t + 2 < t1) prefetch(t + 2);
        }
        if (cas_real) {
          if (item_smem && (a.d_item & 3) == 0 && (reinterpret_cast<uintptr_t>(s_item) & 15) == 0) {
            // shared-memory float adds are CAS loops on sm_100: one 128-bit CAS per 4 columns
            // (quads alternate between the two warp groups)
            uint4* gi = reinterpret_cast<uint4*>(s_item + cas_tile_item * a.d_item);
#pragma unroll
            for (int c = 0; c + 3 < kFP; c += 4) {
              if (c >= a.d_item || ((c >> 2) & 1) != grp) continue;
              uint4* addr = gi + (c >> 2);
              uint4 old = *addr, assumed;
              do {
                assumed = old;
                const uint4 nw = make_uint4(__float_as_uint(__uint_as_float(assumed.x) + df[c]),
                                            __float_as_uint(__uint_as_float(assumed.y) + df[c + 1]),
                                            __float_as_uint(__uint_as_float(assumed.z) + df[c + 2]),
                                            __float_as_uint(__uint_as_float(assumed.w) + df[c + 3]));
                old = sm100::atom_cas128_shared(addr, assumed, nw);
              } while (old.x != assumed.x || old.y != assumed.y || old.z != assumed.z || old.w != assumed.w);
            }
          } else if (item_smem && (a.d_item & 1) == 0) {
            // one 64-bit CAS per column pair (pairs alternate between the two warp groups)
            unsigned long long* gi = reinterpret_cast<unsigned long long*>(s_item + cas_tile_item * a.d_item);
#pragma unroll
            for (int c = 0; c + 1 < kFP; c += 2) {
              if (c >= a.d_item || ((c >> 1) & 1) != grp) continue;
              unsigned long long* addr = gi + (c >> 1);
              unsigned long long old = *addr, assumed;
              do {
                assumed = old;
                const float2 cur = *reinterpret_cast<const float2*>(&assumed);
                const float2 nw = make_float2(cur.x + df[c], cur.y + df[c + 1]);
                old = atomicCAS(addr, assumed, *reinterpret_cast<const unsigned long long*>(&nw));
              } while (old != assumed);
            }
          } else {
            float* gi = (item_smem ? s_item : a.g_item) + cas_tile_item * a.d_item;
#pragma unroll
            for (int c = 0; c < kFP; ++c)
              if (c < a.d_item && (c & 1) == grp) atomicAdd(gi + c, df[c]);
          }
        }
      }
    }
    // ---------------- flush the CTA's accumulators
    if (my_tiles > 0) {
      const int F = a.d_item + a.d_act + a.d_time;
      for (int jh = 0; jh < nh; ++jh) {
        const int f = h0 + 128 * jh + row;                             // hidden unit
        if (grp == 0) {
          float w2[DT];
          tmem_row<DT>(T_DW2 + lane_off + jh * DT, w2);
#pragma unroll
          for (int c = 0; c < DT; ++c) atomicAdd(a.g_seq_w2 + (long long)f * DT + c, w2[c]);
        } else {
          float w1[DT + 16];
          tmem_row<DT + 16>(T_DW1 + lane_off + jh * XK, w1);
#pragma unroll
          for (int c = 0; c < DT; ++c) atomicAdd(a.g_seq_w1 + (long long)c * H2 + f, w1[c]);
          atomicAdd(a.g_seq_b1 + f, w1[DT]);
        }
      }
      if (!last) {
        // the featuriser / table / db2 accumulators belong to the last pass
      } else if (grp == 0) {
        // rows 0..DT-1: [dW_tpᵀ | db_tp]; rows 32..32+DT-1 (the dh half of sDX0): Σ dh (db2)
        float wt[kFP];
        tmem_row<kFP>(T_DWTP + lane_off, wt);                          // warp-collective load
        if (row < DT) {
          for (int k = 0; k < F; ++k) atomicAdd(a.g_tok_w + k * DT + row, wt[k]);
          atomicAdd(a.g_tok_b + row, wt[kFP - 1]);
        } else if (row >= 32 && row < 32 + DT) {
          atomicAdd(a.g_seq_b2 + row - 32, wt[kFP - 1]);
        }
      } else {
        // Y rows: bucket b (0..31) and action 32+a: table grad = Y_row · W_tp[cols]ᵀ
        float y[DT];
        tmem_row<DT>(T_Y + lane_off, y);
        const int e1 = a.d_item, e2 = e1 + a.d_act;
        if (row < a.nb) {
          for (int c = 0; c < a.d_time; ++c) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < DT; ++k) acc = fmaf(y[k], a.tok_w[(e2 + c) * DT + k], acc);
            atomicAdd(a.g_time + row * a.d_time + c, acc);
          }
        } else if (row >= 32 && row < 32 + a.n_actions) {
          for (int c = 0; c < a.d_act; ++c) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < DT; ++k) acc = fmaf(y[k], a.tok_w[(e1 + c) * DT + k], acc);
            atomicAdd(a.g_act + (row - 32) * a.d_act + c, acc);
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (item_smem ? n_item : 0); i += blockDim.x)
    if (s_item[i] != 0.f) atomicAdd(a.g_item + i, s_item[i]);
  for (int i = threadIdx.x; i < kTile * DT; i += blockDim.x) {
    const int rr = i / DT, c = i % DT;
    const int rec = a.Lp - 1 - (cb_last * kTile + rr);
    const float v = s_gpos[rr * (DT + 1) + c];
    if (rec >= 0 && rec < a.L && v != 0.f) atomicAdd(a.g_pos + (long long)rec * DT + c, v);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<512>(tmem);
}

}  // namespace

int frontend_supported(int d, int K, int D, int F, int inner_layers) {
  if (!(d == 16 || d == 32)) return 0;
  if (!(K == 2 || K == 4 || K == 8)) return 0;
  if ((2 * D) % 128 || 2 * D > 512) return 0;
  if (F > kFP - 1) return 0;     // column 31 of the feature tile carries the bias
  if (inner_layers > 8) return 0;
  return 1;
}

int frontend_mlp_bwd_supported(int d, int K, int D) {
  (void)d; (void)K;
  return 2 * D <= 256 || (2 * D) % 256 == 0;
}

int frontend_blob_bytes(int d, int D, int inner_layers) { return blob_offsets(d, D, inner_layers).total * 2; }

void pack_frontend_weights(const float* params, long long tok_w, long long seq_w1, long long seq_w2,
                           const long long (*inner_w)[4], int d, int D, int F, int IL, bf16* blob,
                           const ProjArgs& pj, cudaStream_t st) {
  const BlobOff o = blob_offsets(d, D, IL);
  cudaMemsetAsync(blob, 0, (size_t)o.total * 2, st);
  PackW pw;
  pw.n = 0;
  auto add = [&](long long src, int in, int out, int trans, int n_off, int k_off, int Kdim, int dst, int f16 = 0) {
    auto& s = pw.s[pw.n++];
    s.src = src; s.in = in; s.out = out; s.trans = trans; s.n_off = n_off; s.k_off = k_off; s.Kdim = Kdim; s.dst = dst;
    s.f16 = f16;
  };
  // forward images (Wᵀ, K = in)
  const int XK = d + 16;
  // forward images (Wᵀ, K = in), bias-augmented where the activation tile carries a ones column
  add(tok_w, F, d, 1, 0, 0, kFP, o.tp);
  add(tok_w + (long long)F * d, 1, d, 1, 0, kFP - 1, kFP, o.tp);            // b_tp at k = 31
  add(seq_w1, d, 2 * D, 1, 0, 0, XK, o.w1);
  add(seq_w1 + (long long)d * 2 * D, 1, 2 * D, 1, 0, d, XK, o.w1);          // b1 at k = d
  add(seq_w2, 2 * D, d, 1, 0, 0, 2 * D, o.w2, 1);                           // f16: GELU output operand
  // backward images (W, K = out)
  add(tok_w, F, d, 0, 0, 0, d, o.tp_n);
  add(seq_w1, d, 2 * D, 0, 0, 0, 2 * D, o.w1_n);
  add(seq_w2, 2 * D, d, 0, 0, 0, d, o.w2_n);
  for (int l = 0; l < IL; ++l) {
    const long long wq = inner_w[l][0], wk = inner_w[l][1], wv = inner_w[l][2], wo = inner_w[l][3];
    const long long w1 = wo + (long long)d * d + d, w2 = w1 + 4LL * d * d + 4 * d;   // reference order
    add(wq, d, d, 1, 0, 0, XK, o.qkv[l]);
    add(wk, d, d, 1, d, 0, XK, o.qkv[l]);
    add(wv, d, d, 1, 2 * d, 0, XK, o.qkv[l]);
    add(wq + (long long)d * d, 1, d, 1, 0, d, XK, o.qkv[l]);                 // b_q, b_k, b_v at k = d
    add(wk + (long long)d * d, 1, d, 1, d, d, XK, o.qkv[l]);
    add(wv + (long long)d * d, 1, d, 1, 2 * d, d, XK, o.qkv[l]);
    add(wo, d, d, 1, 0, 0, d, o.wo[l]);
    add(w1, d, 4 * d, 1, 0, 0, XK, o.w1i[l]);
    add(w1 + 4LL * d * d, 1, 4 * d, 1, 0, d, XK, o.w1i[l]);                  // b1 at k = d
    add(w2, 4 * d, d, 1, 0, 0, 4 * d, o.w2i[l], 1);                         // f16: GELU output operand
    add(wq, d, d, 0, 0, 0, 3 * d, o.qkv_n[l]);
    add(wk, d, d, 0, 0, d, 3 * d, o.qkv_n[l]);
    add(wv, d, d, 0, 0, 2 * d, 3 * d, o.qkv_n[l]);
    add(wo, d, d, 0, 0, 0, d, o.wo_n[l]);
    add(w1, d, 4 * d, 0, 0, 0, 4 * d, o.w1i_n[l]);
    add(w2, 4 * d, d, 0, 0, 0, d, o.w2i_n[l]);
  }
  launch(pack_canon_kernel, dim3(16, pw.n + 1), 256, 0, st, params, pw, blob, pj);   // + the table projection
}

template <int DT, int KG, int S>
static int fwd_smem(const FrontArgs& a) {
  const BlobOff bo = blob_offsets(DT, DT * KG, a.inner_layers);
  return ((bo.fwd_total + 63) & ~63) * 2 + S * kTile * (DT + 16 + 64) * 2 +
         (a.inner_layers * 6 * DT + DT + (a.kn_global ? 0 : 2 * DT * KG)) * 4 + (1 + 2 * S) * 8 + 16;
}

template <int DT, int KG, int S>
static int launch_fwd_s(const FrontArgs& a, cudaStream_t st) {
  const int smem = fwd_smem<DT, KG, S>(a);
  smem_attr(fe_fwd_kernel<DT, KG, S>, smem);
  const long long ntiles = (a.T + kTile - 1) / kTile;
  int grid = (int)std::min<long long>((ntiles + S - 1) / S, 148);
  if (g_knobs.fe_grid > 0) grid = std::min(grid, g_knobs.fe_grid);   // testing: many tiles per CTA
  g_launch_fence = kFenceFrontIn | kFenceFrontOut;
  launch(fe_fwd_kernel<DT, KG, S>, grid, 32 * 4 * S, smem, st, a);
  return (int)cudaGetLastError();
}

// as many slots as the weights leave shared memory for (4 at d = 32, D = 128; 3 at D = 256)
template <int DT, int KG>
static int launch_fwd(const FrontArgs& a0, cudaStream_t st) {
  constexpr int kMax = 227 * 1024;
  FrontArgs a = a0;
  a.kn_global = 0;
  if (fwd_smem<DT, KG, 4>(a) <= kMax) return launch_fwd_s<DT, KG, 4>(a, st);
  a.kn_global = g_knobs.fe_kn_global;              // c5 (D = 256): four slots with the LN1 params in L1
  if (a.kn_global && fwd_smem<DT, KG, 4>(a) <= kMax) return launch_fwd_s<DT, KG, 4>(a, st);
  a.kn_global = 0;
  if (fwd_smem<DT, KG, 3>(a) <= kMax) return launch_fwd_s<DT, KG, 3>(a, st);
  if (fwd_smem<DT, KG, 2>(a) <= kMax) return launch_fwd_s<DT, KG, 2>(a, st);
  return (int)cudaErrorInvalidValue;
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

template <int DT>
static int launch_mlp_bwd(const FrontArgs& a, cudaStream_t st) {
  const int H2 = 2 * DT * a.K;
  const int HP = H2 <= 256 ? H2 : 256;            // hidden units per pass
  const int XK = DT + 16;
  const int n_item = a.vocab * a.d_item;
  FrontArgs b = a;
  b.item_smem = g_knobs.item_smem != 0;
  const int tab = (b.item_smem && n_item <= 16384) ? n_item : 0;
  const int smem = (2 * DT * kFP + 2 * HP * DT + HP * XK) * 2 + kTile * (kFP + XK + DT + 128 + 128 + 64 + 64) * 2 +
                   (2 * kTile * (DT + 1) + tab) * 4 + 128;
  if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;
  smem_attr(fe_mlp_bwd_kernel<DT>, 227 * 1024);
  // column-block tiling: grid = tiles-per-sample x replicas (≤ 148 CTAs, one per SM)
  const int tps = (a.Lp + kTile - 1) / kTile;
  int r = std::max(1, std::min(a.B, 148 / tps));
  if (g_knobs.fe_grid > 0) r = std::max(1, std::min(r, g_knobs.fe_grid / tps));   // testing: many tiles per CTA
  int grid = tps * r;
  // split mode: equal ranges of the column-block-major tile order over (up to) every SM — for long
  // sequences (c5: 79 column blocks) one column block per CTA leaves most of the machine idle
  b.mlp_split = 0;
  if (g_knobs.fe_split) {
    const long long W = (long long)tps * a.B;
    int gs = (int)std::min<long long>(W, 148);
    if (g_knobs.fe_grid > 0) gs = std::min(gs, g_knobs.fe_grid);
    const long long col_max = (a.B + r - 1) / r, split_max = (W + gs - 1) / gs;
    // (only for a clear gain: the few SMs column mode leaves free run the side-stream work)
    if (g_knobs.fe_split == 2 || 4 * split_max < 3 * col_max) { b.mlp_split = 1; grid = gs; }
  }
  // > 113 KB of smem keeps one CTA per SM (the kernel allocates all 512 TMEM columns)
  if (H2 <= 256) {
    b.mlp_h0 = 0; b.mlp_hn = 0; b.mlp_last = 1;
    g_launch_fence = kFenceFrontIn | kFenceFrontOut;
    launch(fe_mlp_bwd_kernel<DT>, grid, kThreads8, std::max(smem, 116 * 1024), st, b);
  } else {
    // wider hidden layers: passes of 256 hidden units (TMEM / smem per pass as at 2D = 256), the
    // partial dx0 carried in a.dx0_part; the last pass finishes the featuriser / table part
    if (!a.dx0_part) return (int)cudaErrorInvalidValue;
    for (int h = 0; h < H2; h += HP) {
      b.mlp_h0 = h; b.mlp_hn = HP; b.mlp_last = h + HP >= H2;
      g_launch_fence = kFenceFrontIn | kFenceFrontOut;
      launch(fe_mlp_bwd_kernel<DT>, grid, kThreads8, std::max(smem, 116 * 1024), st, b);
    }
  }
  return (int)cudaGetLastError();
}

int frontend_mlp_bwd(const FrontArgs& a, cudaStream_t st) {
  if (a.d == 32) return launch_mlp_bwd<32>(a, st);
  if (a.d == 16) return launch_mlp_bwd<16>(a, st);
  return (int)cudaErrorInvalidValue;
}

}  // namespace longer
