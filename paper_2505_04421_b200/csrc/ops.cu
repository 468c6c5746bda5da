// ops.cu — SIMT kernels of the LONGER step that are not dense GEMMs: token featurisation,
// layer norms, bias/column reductions, grouped + hybrid attention, global tokens, head + BCE,
// parameter packing and Adam.  Each kernel cites the reference function it restates.
#include "ops.cuh"
#include "sm100.cuh"

#include <math.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace longer {

namespace {
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
}

// ============================================================== front-end: featurisation
// _event_features + abs-pos add (pkg/src/longrec/inputs.py:434-444, :474-476) and the pad
// bookkeeping of encode_events / merge (inputs.py:457-482, merge.py:45-62). One thread/token.
__global__ void embed_fwd_kernel(EmbedArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sw[];                    // tok_w [F*d] + tok_b [d]
  const int F = a.d_item + a.d_act + a.d_time;
  for (int i = threadIdx.x; i < F * a.d + a.d; i += blockDim.x)
    sw[i] = i < F * a.d ? a.tok_w[i] : a.tok_b[i - F * a.d];
  __syncthreads();
  const long long T = (long long)a.B * a.Lp;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int b = (int)(t / a.Lp), j = (int)(t % a.Lp);
  const int n = min(max(a.n_events[b], 0), a.L);
  const bool real = j >= a.Lp - n;
  const int npg = (a.Lp - n) / a.K;
  a.real[t] = real ? 1.f : 0.f;
  a.keep[t] = (j / a.K) >= npg ? 1.f : 0.f;
  if (j == 0) a.npg[b] = npg;
  bf16* fo = a.feat + t * a.FP;
  bf16* xo = a.x0 + t * a.d;
  if (!real) {
    for (int f = 0; f < a.FP; ++f) fo[f] = __float2bfloat16(0.f);
    for (int c = 0; c < a.d; ++c) xo[c] = __float2bfloat16(0.f);
    return;
  }
  const long long src = (long long)b * a.L + (j - (a.Lp - a.L));
  int item = a.items[src], act = a.actions[src], dt = a.dt[src];
  int bad = 0;
  if (item < 0 || item >= a.vocab) { bad |= 1; item = 0; }
  if (act < 0 || act >= a.n_actions) { bad |= 1; act = 0; }
  if (dt < 0) { bad |= 2; dt = 0; }
  if (bad) atomicOr(a.status, bad);
  const int bucket = min(32 - __clz(dt), a.nb - 1);          // time_bucket (inputs.py:307-315)
  const int rec = a.Lp - 1 - j;                              // recency, 0 = most recent
  float feat[64];
  int f = 0;
  for (int c = 0; c < a.d_item; ++c) feat[f++] = a.item_tab[item * a.d_item + c];
  for (int c = 0; c < a.d_act; ++c) feat[f++] = a.act_tab[act * a.d_act + c];
  for (int c = 0; c < a.d_time; ++c) feat[f++] = a.time_tab[bucket * a.d_time + c];
  for (int c = 0; c < a.FP; ++c) fo[c] = __float2bfloat16(c < F ? feat[c] : 0.f);
  const float* pos = a.pos_tab + (long long)rec * a.d;
  for (int c = 0; c < a.d; ++c) {
    float acc = sw[F * a.d + c] + pos[c];
    for (int i = 0; i < F; ++i) acc = fmaf(feat[i], sw[i * a.d + c], acc);
    xo[c] = __float2bfloat16(acc);
  }
}

void embed_fwd(const EmbedArgs& a, cudaStream_t st) {
  const long long T = (long long)a.B * a.Lp;
  const int F = a.d_item + a.d_act + a.d_time;
  const int smem = (F * a.d + a.d) * 4;
  launch(embed_fwd_kernel, cdiv(T, 256), 256, smem, st, a);
}

// Backward of the featuriser (gather_rows bw = np.add.at, tensors.py:505-510): dfeat = dx0·W_tpᵀ
// scattered into the item / action / time tables.  A warp takes one token at a time, lane = channel
// of dx0 (one coalesced row read).  The action and time tables have few rows, so their gradient is
// linear in the per-row SUM of dx0: the block accumulates Σ dx0 per action and per time bucket in
// shared memory (32 lanes → 32 consecutive words, no intra-warp conflicts) and multiplies by W_tpᵀ
// once at the end.  The item part (vocab rows) is a per-token shuffle GEMV against W_tpᵀ in shared
// memory, added into a shared-memory item-gradient copy when the table fits, else into HBM.
constexpr int kEmbedBwdThreads = 256;

__global__ void __launch_bounds__(kEmbedBwdThreads) embed_bwd_kernel(EmbedBwdArgs a, int item_in_smem) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int F = a.d_item + a.d_act + a.d_time, d = a.d;
  float* s_wt = sm;                                  // [d][F]  W_tpᵀ
  float* s_act = s_wt + d * F;                       // [n_actions][d]  Σ dx0 per action
  float* s_time = s_act + a.n_actions * d;           // [nb][d]         Σ dx0 per time bucket
  float* s_item = s_time + a.nb * d;                 // [vocab][d_item] (optional)
  const int n_item = item_in_smem ? a.vocab * a.d_item : 0;
  for (int i = threadIdx.x; i < d * F; i += blockDim.x) s_wt[(i % d) * F + i / d] = a.tok_w[i];
  for (int i = threadIdx.x; i < (a.n_actions + a.nb) * d + n_item; i += blockDim.x) s_act[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = blockDim.x / 32;
  const long long T = (long long)a.B * a.Lp;
  for (long long t = (long long)blockIdx.x * nw + threadIdx.x / 32; t < T; t += (long long)gridDim.x * nw) {
    const int b = (int)(t / a.Lp), j = (int)(t % a.Lp);
    const int n = min(max(a.n_events[b], 0), a.L);
    if (j < a.Lp - n) continue;
    const long long src = (long long)b * a.L + (j - (a.Lp - a.L));
    int item = a.items[src], act = a.actions[src], dt = a.dt[src];
    if (item < 0 || item >= a.vocab) item = 0;
    if (act < 0 || act >= a.n_actions) act = 0;
    if (dt < 0) dt = 0;
    const int bucket = min(32 - __clz(dt), a.nb - 1);
    const float* dx = a.dx0 + t * d;
    const float v0 = lane < d ? dx[lane] : 0.f;
    const float v1 = lane + 32 < d ? dx[lane + 32] : 0.f;
    if (lane < d) {
      atomicAdd(&s_act[act * d + lane], v0);
      atomicAdd(&s_time[bucket * d + lane], v0);
    }
    if (lane + 32 < d) {
      atomicAdd(&s_act[act * d + lane + 32], v1);
      atomicAdd(&s_time[bucket * d + lane + 32], v1);
    }
    for (int f0 = 0; f0 < a.d_item; f0 += 32) {
      const int fi = f0 + lane;
      const int fc = min(fi, F - 1);
      float g = 0.f;
#pragma unroll 8
      for (int c = 0; c < min(d, 32); ++c) g = fmaf(__shfl_sync(0xffffffffu, v0, c), s_wt[c * F + fc], g);
      for (int c = 32; c < d; ++c) g = fmaf(__shfl_sync(0xffffffffu, v1, c - 32), s_wt[c * F + fc], g);
      if (fi < a.d_item) {
        if (item_in_smem) atomicAdd(&s_item[item * a.d_item + fi], g);
        else atomicAdd(&a.g_item[(long long)item * a.d_item + fi], g);
      }
    }
  }
  __syncthreads();
  // g_act[r, f] += Σ_c S_act[r, c]·W_tp[d_item + f, c]; likewise the time rows
  for (int i = threadIdx.x; i < a.n_actions * a.d_act + a.nb * a.d_time; i += blockDim.x) {
    const bool is_act = i < a.n_actions * a.d_act;
    const int k = is_act ? i : i - a.n_actions * a.d_act;
    const int w = is_act ? a.d_act : a.d_time;
    const int r = k / w, f = (is_act ? a.d_item : a.d_item + a.d_act) + k % w;
    const float* S = (is_act ? s_act : s_time) + r * d;
    float g = 0.f;
    for (int c = 0; c < d; ++c) g = fmaf(S[c], s_wt[c * F + f], g);
    if (g != 0.f) atomicAdd(is_act ? &a.g_act[k] : &a.g_time[k], g);
  }
  for (int i = threadIdx.x; i < n_item; i += blockDim.x)
    if (s_item[i] != 0.f) atomicAdd(&a.g_item[i], s_item[i]);
}

// abs_pos_table gradient: row r collects dx0 of the token with recency r of every sample —
// a deterministic strided column reduction instead of scatter atomics.
__global__ void pos_grad_kernel(EmbedBwdArgs a) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;                     // recency row
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
    float acc = 0.f;
    for (int b = 0; b < a.B; ++b) {
      const int n = min(max(a.n_events[b], 0), a.L);
      if (r < n) acc += a.dx0[((long long)b * a.Lp + (a.Lp - 1 - r)) * a.d + c];
    }
    a.g_pos[(long long)r * a.d + c] += acc;
  }
}

void embed_bwd(const EmbedBwdArgs& a, cudaStream_t st) {
  const long long T = (long long)a.B * a.Lp;
  const int F = a.d_item + a.d_act + a.d_time;
  if (a.d > 64) { fprintf(stderr, "embed_bwd: d = %d > 64 not supported\n", a.d); abort(); }
  const int base = 4 * (F * a.d + (a.n_actions + a.nb) * a.d);
  const int item_in_smem = (base + 4LL * a.vocab * a.d_item <= 64 * 1024) ? 1 : 0;
  const int smem = base + (item_in_smem ? 4 * a.vocab * a.d_item : 0);
  smem_attr(embed_bwd_kernel, smem);
  const int grid = (int)std::min<long long>(cdiv(T, kEmbedBwdThreads / 32), 148 * 4);
  launch(embed_bwd_kernel, grid, kEmbedBwdThreads, smem, st, a, item_in_smem);
  launch(pos_grad_kernel, a.L, 32 * cdiv(a.d, 32), 0, st, a);
}

// ============================================================== layer norm
// One warp per row.  Contiguous mode (W == 32·VPT, aligned rows): lane owns columns
// [lane·VPT, lane·VPT + VPT) and moves them with one 8/16/32-byte access; otherwise strided.
template <int VPT, bool CONTIG>
__device__ __forceinline__ int ln_col(int lane, int u) { return CONTIG ? lane * VPT + u : lane + 32 * u; }

template <int VPT, bool CONTIG>
__device__ __forceinline__ void ln_load(const float* __restrict__ p, int lane, int W, float* v) {
  if constexpr (CONTIG && VPT == 8) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p + lane * 8));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + lane * 8 + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else if constexpr (CONTIG && VPT == 4) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p + lane * 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else if constexpr (CONTIG && VPT == 2) {
    const float2 a = __ldg(reinterpret_cast<const float2*>(p + lane * 2));
    v[0] = a.x; v[1] = a.y;
  } else {
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int c = ln_col<VPT, CONTIG>(lane, u);
      v[u] = c < W ? p[c] : 0.f;
    }
  }
}

template <int VPT, bool CONTIG>
__device__ __forceinline__ void ln_load(const bf16* __restrict__ p, int lane, int W, float* v) {
  if constexpr (CONTIG && VPT == 8) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p + lane * 8));
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) { v[2 * t] = sm100::bf16_lo(w[t]); v[2 * t + 1] = sm100::bf16_hi(w[t]); }
  } else if constexpr (CONTIG && VPT == 4) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(p + lane * 4));
    v[0] = sm100::bf16_lo(a.x); v[1] = sm100::bf16_hi(a.x); v[2] = sm100::bf16_lo(a.y); v[3] = sm100::bf16_hi(a.y);
  } else {
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int c = ln_col<VPT, CONTIG>(lane, u);
      v[u] = c < W ? __bfloat162float(p[c]) : 0.f;
    }
  }
}

template <int VPT, bool CONTIG>
__global__ void ln_fwd_kernel(RowMap x, int W, const float* __restrict__ g, const float* __restrict__ bta,
                              bf16* y, float* mean, float* rstd, float* xcopy) {
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= x.rows()) return;
  const int per = x.na + x.nb;
  const int b = row / per, j = row % per;
  const float* src = j < x.na ? x.A + (long long)(b * x.a_rows + x.a_off + j) * x.lda
                              : x.Bsrc + (long long)(b * x.nb + j - x.na) * x.ldb;
  float v[VPT];
  ln_load<VPT, CONTIG>(src, lane, W, v);
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < VPT; ++u) s += v[u];
  const float mu = warp_sum(s) / W;
  float q = 0.f;
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const int c = ln_col<VPT, CONTIG>(lane, u);
    const float dv = c < W ? v[u] - mu : 0.f;
    q += dv * dv;
  }
  const float var = warp_sum(q) / W;
  const float inv = rsqrtf(var + kLnEps);
  const int orow = x.out_row(row);
  bf16* dst = y + (long long)orow * W;
  if (xcopy) {                                        // the gathered input rows, materialised
    float* xc = xcopy + (long long)orow * W;
    if constexpr (CONTIG && VPT == 4) {
      *reinterpret_cast<float4*>(xc + lane * 4) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int c = ln_col<VPT, CONTIG>(lane, u);
        if (c < W) xc[c] = v[u];
      }
    }
  }
  if constexpr (CONTIG && VPT >= 2) {
    float gg[VPT], bb[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) { gg[u] = g[lane * VPT + u]; bb[u] = bta[lane * VPT + u]; }
    uint32_t w[VPT / 2];
#pragma unroll
    for (int u = 0; u < VPT; u += 2)
      w[u / 2] = sm100::pack_bf16((v[u] - mu) * inv * gg[u] + bb[u], (v[u + 1] - mu) * inv * gg[u + 1] + bb[u + 1]);
    if constexpr (VPT == 8) *reinterpret_cast<uint4*>(dst + lane * 8) = make_uint4(w[0], w[1], w[2], w[3]);
    else if constexpr (VPT == 4) *reinterpret_cast<uint2*>(dst + lane * 4) = make_uint2(w[0], w[1]);
    else *reinterpret_cast<uint32_t*>(dst + lane * 2) = w[0];
  } else {
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int c = ln_col<VPT, CONTIG>(lane, u);
      if (c < W) dst[c] = __float2bfloat16((v[u] - mu) * inv * g[c] + bta[c]);
    }
  }
  if (lane == 0) { mean[orow] = mu; rstd[orow] = inv; }
}

namespace {
bool ln_contig(int W, int vpt, const void* p0, int ld0, const void* p1, int ld1) {
  if (W != 32 * vpt || vpt == 1) return false;
  auto al = [&](const void* p, int ld) {
    return !p || ((reinterpret_cast<uintptr_t>(p) % (4 * vpt)) == 0 && ld % vpt == 0);
  };
  return al(p0, ld0) && al(p1, ld1);
}
}  // namespace

void layernorm_fwd(const RowMap& x, int W, const float* g, const float* b, bf16* y, float* mean, float* rstd,
                   cudaStream_t st, float* xcopy) {
  const int rows = x.rows();
  if (rows <= 0) return;
  const int grid = cdiv(rows, 8);
  const int vpt = W <= 32 ? 1 : W <= 64 ? 2 : W <= 128 ? 4 : 8;
  const bool ct = ln_contig(W, vpt, x.A, x.lda, x.nb ? x.Bsrc : nullptr, x.ldb);
#define LNF(V) (ct ? launch(ln_fwd_kernel<V, true>, grid, 256, 0, st, x, W, g, b, y, mean, rstd, xcopy) \
                   : launch(ln_fwd_kernel<V, false>, grid, 256, 0, st, x, W, g, b, y, mean, rstd, xcopy))
  if (vpt == 1) launch(ln_fwd_kernel<1, false>, grid, 256, 0, st, x, W, g, b, y, mean, rstd, xcopy);
  else if (vpt == 2) LNF(2);
  else if (vpt == 4) LNF(4);
  else LNF(8);
#undef LNF
}

// LN backward (pkg/src/longrec/tensors.py:368-378): dx = (ĝ − mean ĝ − x̂·mean(ĝx̂))·σ⁻¹, ĝ = dy·g
template <int VPT, bool CONTIG, typename TY = float>
__global__ void ln_bwd_kernel(RowMap x, int W, const float* __restrict__ g, const float* __restrict__ mean,
                              const float* __restrict__ rstd, const TY* __restrict__ dy, int ldy, RowMapW out,
                              int accumulate, const float* rowmask, float* dgain, float* dbias, LnBwdExtra ex) {
  pdl_trigger();
  pdl_wait();
  __shared__ float sg[8][VPT * 32], sb[8][VPT * 32], sc[8][VPT * 32];
  const int warps = blockDim.x / 32;
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int rows = x.rows();
  const int per = x.na + x.nb;
  float pg[VPT], pb[VPT], pc[VPT], gv[VPT];
#pragma unroll
  for (int u = 0; u < VPT; ++u) { pg[u] = 0.f; pb[u] = 0.f; pc[u] = 0.f; }
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const int c = ln_col<VPT, CONTIG>(lane, u);
    gv[u] = c < W ? g[c] : 0.f;
  }
  // software-pipelined over the warp's rows: the inputs of the next rows are loaded before row r
  // is reduced and stored
  struct RowIn {
    float x[VPT], dy[VPT], o[VPT], ad[VPT];
    float mu, inv, rm;
    float* dst;
  };
  auto load_row = [&](int row, RowIn& R) {
    const int b = row / per, j = row % per;
    const float* src = j < x.na ? x.A + (long long)(b * x.a_rows + x.a_off + j) * x.lda
                                : x.Bsrc + (long long)(b * x.nb + j - x.na) * x.ldb;
    R.dst = j < out.na ? out.A + (long long)(b * out.a_rows + out.a_off + j) * out.lda
                       : out.Bsrc + (long long)(b * out.nb + j - out.na) * out.ldb;
    R.mu = mean[row];
    R.inv = rstd[row];
    R.rm = rowmask ? rowmask[row] : 1.f;
    ln_load<VPT, CONTIG>(src, lane, W, R.x);
    ln_load<VPT, CONTIG>(dy + (long long)row * ldy, lane, W, R.dy);
    if (accumulate) ln_load<VPT, CONTIG>(R.dst, lane, W, R.o);
    if (ex.addend) ln_load<VPT, CONTIG>(ex.addend + (long long)row * W, lane, W, R.ad);
  };
  const int stride = gridDim.x * warps;
  int row = blockIdx.x * warps + wid;
  // VPT ≤ 4: three rows in flight (the warp's next two rows load while this one is reduced)
  constexpr bool DEEP = VPT <= 4;
  RowIn cur, nxt;
  if (row < rows) load_row(row, cur);
  if (DEEP && row + stride < rows) load_row(row + stride, nxt);
  for (; row < rows; row += stride) {
    RowIn nn;
    if (DEEP) {
      if (row + 2 * stride < rows) load_row(row + 2 * stride, nn);
    } else if (row + stride < rows) {
      load_row(row + stride, nxt);
    }
    const float mu = cur.mu, inv = cur.inv, rm = cur.rm;
    float* dst = cur.dst;
    float xh[VPT], gh[VPT], dyv[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) { xh[u] = cur.x[u]; dyv[u] = cur.dy[u]; }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int c = ln_col<VPT, CONTIG>(lane, u);
      if (c < W) {
        xh[u] = (xh[u] - mu) * inv;
        gh[u] = dyv[u] * gv[u];
        pg[u] += dyv[u] * xh[u];
        pb[u] += dyv[u];
      } else {
        xh[u] = 0.f; gh[u] = 0.f;
      }
      s1 += gh[u];
      s2 += gh[u] * xh[u];
    }
    const float m1 = warp_sum(s1) / W, m2 = warp_sum(s2) / W;
    float o[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      float v = (gh[u] - m1 - xh[u] * m2) * inv;
      if (accumulate) v += cur.o[u];
      if (ex.addend) v += cur.ad[u];
      o[u] = v * rm;
      pc[u] += o[u];
    }
    if (ex.out_bf) {
      bf16* ob = ex.out_bf + (long long)row * W;
      if constexpr (CONTIG && VPT >= 2) {
        uint32_t w[VPT / 2];
#pragma unroll
        for (int u = 0; u < VPT; u += 2) w[u / 2] = sm100::pack_bf16(o[u], o[u + 1]);
        if constexpr (VPT == 8) *reinterpret_cast<uint4*>(ob + lane * 8) = make_uint4(w[0], w[1], w[2], w[3]);
        else if constexpr (VPT == 4) *reinterpret_cast<uint2*>(ob + lane * 4) = make_uint2(w[0], w[1]);
        else *reinterpret_cast<uint32_t*>(ob + lane * 2) = w[0];
      } else {
#pragma unroll
        for (int u = 0; u < VPT; ++u) {
          const int c = ln_col<VPT, CONTIG>(lane, u);
          if (c < W) ob[c] = __float2bfloat16(o[u]);
        }
      }
    }
    if constexpr (CONTIG && VPT == 8) {
      reinterpret_cast<float4*>(dst + lane * 8)[0] = make_float4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<float4*>(dst + lane * 8)[1] = make_float4(o[4], o[5], o[6], o[7]);
    } else if constexpr (CONTIG && VPT == 4) {
      *reinterpret_cast<float4*>(dst + lane * 4) = make_float4(o[0], o[1], o[2], o[3]);
    } else if constexpr (CONTIG && VPT == 2) {
      *reinterpret_cast<float2*>(dst + lane * 2) = make_float2(o[0], o[1]);
    } else {
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int c = ln_col<VPT, CONTIG>(lane, u);
        if (c < W) dst[c] = o[u];
      }
    }
    cur = nxt;
    if (DEEP) nxt = nn;
  }
  if (dgain || ex.colsum_out) {
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int c = ln_col<VPT, CONTIG>(lane, u);
      sg[wid][c] = pg[u]; sb[wid][c] = pb[u]; sc[wid][c] = pc[u];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
      float a = 0.f, bb = 0.f, cc = 0.f;
      for (int w = 0; w < warps; ++w) { a += sg[w][c]; bb += sb[w][c]; cc += sc[w][c]; }
      if (dgain) { atomicAdd(&dgain[c], a); atomicAdd(&dbias[c], bb); }
      if (ex.colsum_out) atomicAdd(&ex.colsum_out[c], cc);
    }
  }
}

// Pipelined lean LN backward (W = 128, bf16 dy, no extras): each warp streams its rows through an
// S-stage ring of shared memory with per-lane cp.async (16 B of x, 8 B of dy per lane and row, the
// row statistics by lanes 0..R-1), so S-1 groups of R rows stay in flight while the current group
// is reduced — deep memory-level parallelism without holding the rows in registers.
__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cpa4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g));
}
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int R, int S>
struct LnAsync {
  static constexpr int STAGE = R * 768 + 32 * 4;   // x rows fp32 | dy rows bf16 | mean[R], rstd[R]
  static constexpr int SMEM = 8 * S * STAGE;
};

// Half-warp-per-row variant: 16 lanes × 8 columns per row, the two half-warps on neighbouring rows,
// so every address computation, shuffle and loop step covers two rows (R = rows per stage, even).
template <int R, int S>
__global__ void __launch_bounds__(256) ln_bwd128_hw_kernel(RowMap x, const float* __restrict__ g,
                                                           const float* __restrict__ mean,
                                                           const float* __restrict__ rstd,
                                                           const bf16* __restrict__ dy, int ldy, RowMapW out,
                                                           float* dgain, float* dbias) {
  pdl_trigger();
  pdl_wait();
  using L = LnAsync<R, S>;
  extern __shared__ __align__(16) uint8_t lsm[];
  __shared__ float sg[16][128], sb[16][128];
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, h = lane >> 4, l = lane & 15;
  uint8_t* wbase = lsm + wid * S * L::STAGE;
  const int rows = x.rows();
  const int per = x.na + x.nb;
  float gg[8];
  {
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(g) + 2 * l);
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(g) + 2 * l + 1);
    gg[0] = g0.x; gg[1] = g0.y; gg[2] = g0.z; gg[3] = g0.w; gg[4] = g1.x; gg[5] = g1.y; gg[6] = g1.z; gg[7] = g1.w;
  }
  float pg[8], pb[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) { pg[u] = 0.f; pb[u] = 0.f; }
  const int stride = gridDim.x * 8 * R;
  const int first = (blockIdx.x * 8 + wid) * R;
  const float inv_per = 1.f / (float)per;
  auto split = [&](int row, int& b, int& j) {
    b = (int)(((float)row + 0.5f) * inv_per);
    j = row - b * per;
    if (j < 0) { --b; j += per; } else if (j >= per) { ++b; j -= per; }
  };
  auto issue = [&](int r0, int s) {
    uint8_t* sp = wbase + s * L::STAGE;
    float* sx = reinterpret_cast<float*>(sp);
    bf16* sd = reinterpret_cast<bf16*>(sp + R * 512);
    float* ss = reinterpret_cast<float*>(sp + R * 768);
#pragma unroll
    for (int i = 0; i < R; i += 2) {
      const int row = r0 + i + h;
      if (row < rows) {
        int b, j;
        split(row, b, j);
        const float* src = j < x.na ? x.A + (long long)(b * x.a_rows + x.a_off + j) * x.lda
                                    : x.Bsrc + (long long)(b * x.nb + j - x.na) * x.ldb;
        cpa16(sx + (i + h) * 128 + l * 8, src + l * 8);
        cpa16(sx + (i + h) * 128 + l * 8 + 4, src + l * 8 + 4);
        cpa16(sd + (i + h) * 128 + l * 8, dy + (long long)row * ldy + l * 8);
      }
    }
    if (lane < R && r0 + lane < rows) {
      cpa4(ss + lane, mean + r0 + lane);
      cpa4(ss + R + lane, rstd + r0 + lane);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(first + s * stride, s);
  int it = 0;
  for (int r0 = first; r0 < rows; r0 += stride, ++it) {
    __syncwarp();
    issue(r0 + (S - 1) * stride, (it + S - 1) % S);
    cpa_wait<S - 1>();
    __syncwarp();
    const uint8_t* sp = wbase + (it % S) * L::STAGE;
    const float* sx = reinterpret_cast<const float*>(sp);
    const bf16* sd = reinterpret_cast<const bf16*>(sp + R * 512);
    const float* ss = reinterpret_cast<const float*>(sp + R * 768);
#pragma unroll
    for (int i = 0; i < R; i += 2) {
      if (r0 + i >= rows) break;                   // warp-uniform
      const int row = r0 + i + h;
      const bool valid = row < rows;
      float xr[8], d[8];
      const float4 x0 = *reinterpret_cast<const float4*>(sx + (i + h) * 128 + l * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(sx + (i + h) * 128 + l * 8 + 4);
      const uint4 dv = *reinterpret_cast<const uint4*>(sd + (i + h) * 128 + l * 8);
      xr[0] = x0.x; xr[1] = x0.y; xr[2] = x0.z; xr[3] = x0.w; xr[4] = x1.x; xr[5] = x1.y; xr[6] = x1.z; xr[7] = x1.w;
      d[0] = sm100::bf16_lo(dv.x); d[1] = sm100::bf16_hi(dv.x); d[2] = sm100::bf16_lo(dv.y); d[3] = sm100::bf16_hi(dv.y);
      d[4] = sm100::bf16_lo(dv.z); d[5] = sm100::bf16_hi(dv.z); d[6] = sm100::bf16_lo(dv.w); d[7] = sm100::bf16_hi(dv.w);
      const float mu = valid ? ss[i + h] : 0.f, inv = valid ? ss[R + i + h] : 0.f;
      if (!valid) {
#pragma unroll
        for (int u = 0; u < 8; ++u) { xr[u] = 0.f; d[u] = 0.f; }
      }
      float xh[8], gh[8], s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xh[u] = (xr[u] - mu) * inv;
        gh[u] = d[u] * gg[u];
        s1 += gh[u];
        s2 += gh[u] * xh[u];
        pg[u] += d[u] * xh[u];
        pb[u] += d[u];
      }
      // per half-warp: lanes l < 8 end with the row's s1, lanes l ≥ 8 with its s2
      float kp = (l & 8) ? s2 : s1;
      kp += __shfl_xor_sync(0xffffffffu, (l & 8) ? s1 : s2, 8);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) kp += __shfl_xor_sync(0xffffffffu, kp, o);
      const float m1 = __shfl_sync(0xffffffffu, kp, h * 16) * (1.f / 128);
      const float m2 = __shfl_sync(0xffffffffu, kp, h * 16 + 8) * (1.f / 128);
      if (valid) {
        int b, j;
        split(row, b, j);
        float* dst = j < out.na ? out.A + (long long)(b * out.a_rows + out.a_off + j) * out.lda
                                : out.Bsrc + (long long)(b * out.nb + j - out.na) * out.ldb;
        float o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) o[u] = (gh[u] - m1 - xh[u] * m2) * inv;
        reinterpret_cast<float4*>(dst + l * 8)[0] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(dst + l * 8)[1] = make_float4(o[4], o[5], o[6], o[7]);
      }
    }
  }
  cpa_wait<0>();
#pragma unroll
  for (int u = 0; u < 8; ++u) { sg[wid * 2 + h][l * 8 + u] = pg[u]; sb[wid * 2 + h][l * 8 + u] = pb[u]; }
  __syncthreads();
  if (threadIdx.x < 128) {
    float a = 0.f, bb = 0.f;
#pragma unroll
    for (int w = 0; w < 16; ++w) { a += sg[w][threadIdx.x]; bb += sb[w][threadIdx.x]; }
    if (dgain) { atomicAdd(&dgain[threadIdx.x], a); atomicAdd(&dbias[threadIdx.x], bb); }
  }
}

// The same pipeline at W = 256 (c5's K/V rows): a full warp per row, 8 columns per lane, R rows per
// stage (x fp32 | dy bf16 | mean, rstd), S stages per warp.
template <int R, int S>
struct LnAsync256 {
  static constexpr int STAGE = R * 1536 + 32 * 4;
  static constexpr int SMEM = 8 * S * STAGE;
};

template <int R, int S>
__global__ void __launch_bounds__(256) ln_bwd256_kernel(RowMap x, const float* __restrict__ g,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        const bf16* __restrict__ dy, int ldy, RowMapW out,
                                                        float* dgain, float* dbias) {
  pdl_trigger();
  pdl_wait();
  using L = LnAsync256<R, S>;
  extern __shared__ __align__(16) uint8_t lsm[];
  __shared__ float sg[8][256], sb[8][256];
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint8_t* wbase = lsm + wid * S * L::STAGE;
  const int rows = x.rows();
  const int per = x.na + x.nb;
  float gg[8];
  {
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(g) + 2 * lane);
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(g) + 2 * lane + 1);
    gg[0] = g0.x; gg[1] = g0.y; gg[2] = g0.z; gg[3] = g0.w; gg[4] = g1.x; gg[5] = g1.y; gg[6] = g1.z; gg[7] = g1.w;
  }
  float pg[8], pb[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) { pg[u] = 0.f; pb[u] = 0.f; }
  const int stride = gridDim.x * 8 * R;
  const int first = (blockIdx.x * 8 + wid) * R;
  const float inv_per = 1.f / (float)per;
  auto split = [&](int row, int& b, int& j) {
    b = (int)(((float)row + 0.5f) * inv_per);
    j = row - b * per;
    if (j < 0) { --b; j += per; } else if (j >= per) { ++b; j -= per; }
  };
  auto issue = [&](int r0, int s) {
    uint8_t* sp = wbase + s * L::STAGE;
    float* sx = reinterpret_cast<float*>(sp);
    bf16* sd = reinterpret_cast<bf16*>(sp + R * 1024);
    float* ss = reinterpret_cast<float*>(sp + R * 1536);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = r0 + i;
      if (row < rows) {
        int b, j;
        split(row, b, j);
        const float* src = j < x.na ? x.A + (long long)(b * x.a_rows + x.a_off + j) * x.lda
                                    : x.Bsrc + (long long)(b * x.nb + j - x.na) * x.ldb;
        cpa16(sx + i * 256 + lane * 8, src + lane * 8);
        cpa16(sx + i * 256 + lane * 8 + 4, src + lane * 8 + 4);
        cpa16(sd + i * 256 + lane * 8, dy + (long long)row * ldy + lane * 8);
      }
    }
    if (lane < R && r0 + lane < rows) {
      cpa4(ss + lane, mean + r0 + lane);
      cpa4(ss + R + lane, rstd + r0 + lane);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) issue(first + s * stride, s);
  int it = 0;
  for (int r0 = first; r0 < rows; r0 += stride, ++it) {
    __syncwarp();
    issue(r0 + (S - 1) * stride, (it + S - 1) % S);
    cpa_wait<S - 1>();
    __syncwarp();
    const uint8_t* sp = wbase + (it % S) * L::STAGE;
    const float* sx = reinterpret_cast<const float*>(sp);
    const bf16* sd = reinterpret_cast<const bf16*>(sp + R * 1024);
    const float* ss = reinterpret_cast<const float*>(sp + R * 1536);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = r0 + i;
      if (row >= rows) break;                      // warp-uniform
      float xr[8], d[8];
      const float4 x0 = *reinterpret_cast<const float4*>(sx + i * 256 + lane * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(sx + i * 256 + lane * 8 + 4);
      const uint4 dv = *reinterpret_cast<const uint4*>(sd + i * 256 + lane * 8);
      xr[0] = x0.x; xr[1] = x0.y; xr[2] = x0.z; xr[3] = x0.w; xr[4] = x1.x; xr[5] = x1.y; xr[6] = x1.z; xr[7] = x1.w;
      d[0] = sm100::bf16_lo(dv.x); d[1] = sm100::bf16_hi(dv.x); d[2] = sm100::bf16_lo(dv.y); d[3] = sm100::bf16_hi(dv.y);
      d[4] = sm100::bf16_lo(dv.z); d[5] = sm100::bf16_hi(dv.z); d[6] = sm100::bf16_lo(dv.w); d[7] = sm100::bf16_hi(dv.w);
      const float mu = ss[i], inv = ss[R + i];
      float xh[8], gh[8], s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xh[u] = (xr[u] - mu) * inv;
        gh[u] = d[u] * gg[u];
        s1 += gh[u];
        s2 += gh[u] * xh[u];
        pg[u] += d[u] * xh[u];
        pb[u] += d[u];
      }
      // lanes < 16 end with the row's s1, lanes >= 16 with its s2
      float kp = (lane & 16) ? s2 : s1;
      kp += __shfl_xor_sync(0xffffffffu, (lane & 16) ? s1 : s2, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) kp += __shfl_xor_sync(0xffffffffu, kp, o);
      const float m1 = __shfl_sync(0xffffffffu, kp, 0) * (1.f / 256);
      const float m2 = __shfl_sync(0xffffffffu, kp, 16) * (1.f / 256);
      int b, j;
      split(row, b, j);
      float* dst = j < out.na ? out.A + (long long)(b * out.a_rows + out.a_off + j) * out.lda
                              : out.Bsrc + (long long)(b * out.nb + j - out.na) * out.ldb;
      float o[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) o[u] = (gh[u] - m1 - xh[u] * m2) * inv;
      reinterpret_cast<float4*>(dst + lane * 8)[0] = make_float4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<float4*>(dst + lane * 8)[1] = make_float4(o[4], o[5], o[6], o[7]);
    }
  }
  cpa_wait<0>();
#pragma unroll
  for (int u = 0; u < 8; ++u) { sg[wid][lane * 8 + u] = pg[u]; sb[wid][lane * 8 + u] = pb[u]; }
  __syncthreads();
  {
    float a = 0.f, bb = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) { a += sg[w][threadIdx.x]; bb += sb[w][threadIdx.x]; }
    if (dgain) { atomicAdd(&dgain[threadIdx.x], a); atomicAdd(&dbias[threadIdx.x], bb); }
  }
}

template <int R, int S>
static void launch_ln256(int bps, const RowMap& x, const float* g, const float* mean, const float* rstd,
                         const bf16* dy, int ldy, const RowMapW& out, float* dgain, float* dbias, cudaStream_t st) {
  constexpr int smem = LnAsync256<R, S>::SMEM;
  smem_attr(ln_bwd256_kernel<R, S>, smem);
  const int grid = std::max(1, std::min(cdiv(x.rows(), 8 * R), 148 * bps));
  launch(ln_bwd256_kernel<R, S>, grid, 256, smem, st, x, g, mean, rstd, dy, ldy, out, dgain, dbias);
}

template <int R, int S>
static void launch_ln_hw(int bps, const RowMap& x, const float* g, const float* mean, const float* rstd,
                         const bf16* dy, int ldy, const RowMapW& out, float* dgain, float* dbias, cudaStream_t st) {
  constexpr int smem = LnAsync<R, S>::SMEM;
  smem_attr(ln_bwd128_hw_kernel<R, S>, smem);
  const int grid = std::max(1, std::min(cdiv(x.rows(), 8 * R), 148 * bps));
  launch(ln_bwd128_hw_kernel<R, S>, grid, 256, smem, st, x, g, mean, rstd, dy, ldy, out, dgain, dbias);
}

// bf16 dy (a dX GEMM written in bf16: half the bytes of the HBM-bound K/V-row LN backward)
void layernorm_bwd(const RowMap& x, int W, const float* g, const float* mean, const float* rstd, const bf16* dy,
                   int ldy, const RowMapW& out, float* dgain, float* dbias, cudaStream_t st) {
  const int rows = x.rows();
  if (rows <= 0) return;
  const int grid = std::max(1, std::min(cdiv(rows, 32), 148 * 8));
  const bool ct = W == 128 && ln_contig(W, 4, x.A, x.lda, x.nb ? x.Bsrc : nullptr, x.ldb) &&
                  ln_contig(W, 4, out.A, out.lda, out.nb ? out.Bsrc : nullptr, out.ldb) && ldy % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(dy) & 7) == 0;
  const bool dy16 = ldy % 8 == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0 &&   // 16-byte dy rows,
                    (reinterpret_cast<uintptr_t>(g) & 15) == 0;                      // float4 gains
  const bool ct256 = W == 256 && ln_contig(W, 8, x.A, x.lda, x.nb ? x.Bsrc : nullptr, x.ldb) &&
                     ln_contig(W, 8, out.A, out.lda, out.nb ? out.Bsrc : nullptr, out.ldb);
  if (ct && dy16) {
    launch_ln_hw<4, 3>(2, x, g, mean, rstd, dy, ldy, out, dgain, dbias, st);
  } else if (ct256 && dy16 && g_knobs.ln256) {
    launch_ln256<4, 3>(1, x, g, mean, rstd, dy, ldy, out, dgain, dbias, st);
  } else if (ct)
    launch(ln_bwd_kernel<4, true, bf16>, grid, 256, 0, st, x, W, g, mean, rstd, dy, ldy, out, 0,
           static_cast<const float*>(nullptr), dgain, dbias, LnBwdExtra());
  else if (W <= 128)
    launch(ln_bwd_kernel<4, false, bf16>, grid, 256, 0, st, x, W, g, mean, rstd, dy, ldy, out, 0,
           static_cast<const float*>(nullptr), dgain, dbias, LnBwdExtra());
  else
    launch(ln_bwd_kernel<8, false, bf16>, grid, 256, 0, st, x, W, g, mean, rstd, dy, ldy, out, 0,
           static_cast<const float*>(nullptr), dgain, dbias, LnBwdExtra());
}

void layernorm_bwd(const RowMap& x, int W, const float* g, const float* mean, const float* rstd, const float* dy,
                   int ldy, const RowMapW& out, int accumulate, const float* rowmask, float* dgain, float* dbias,
                   cudaStream_t st, LnBwdExtra ex) {
  const int rows = x.rows();
  if (rows <= 0) return;
  // ~32 rows per 8-warp block: enough blocks to cover the SMs, few enough that the per-block
  // atomic flush of the column partials stays cheap
  constexpr int rpb = 32;                      // 8 / 16 / 64 measured slower (round 1)
  const int grid = std::max(1, std::min(cdiv(rows, rpb), 148 * 8));
  const int vpt = W <= 32 ? 1 : W <= 64 ? 2 : W <= 128 ? 4 : 8;
  const bool ct = ln_contig(W, vpt, x.A, x.lda, x.nb ? x.Bsrc : nullptr, x.ldb) &&
                  ln_contig(W, vpt, out.A, out.lda, out.nb ? out.Bsrc : nullptr, out.ldb) &&
                  ln_contig(W, vpt, dy, ldy, nullptr, 0);

#define LNB(V) (ct ? launch(ln_bwd_kernel<V, true>, grid, 256, 0, st, x, W, g, mean, rstd, dy, ldy, out, accumulate, rowmask, dgain, dbias, ex) \
                   : launch(ln_bwd_kernel<V, false>, grid, 256, 0, st, x, W, g, mean, rstd, dy, ldy, out, accumulate, rowmask, dgain, dbias, ex))
  if (vpt == 1) launch(ln_bwd_kernel<1, false>, grid, 256, 0, st, x, W, g, mean, rstd, dy, ldy, out, accumulate, rowmask, dgain, dbias, ex);
  else if (vpt == 2) LNB(2);
  else if (vpt == 4) LNB(4);
  else LNB(8);
#undef LNB
}

// ============================================================== reductions / copies
template <typename T>
__global__ void colsum_kernel(const T* __restrict__ x, int rows, int W, int ld, int rows_per_block, float* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[256];
  const int cpp = W < 256 ? W : 256;
  const int rpp = 256 / cpp;
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  for (int c0 = 0; c0 < W; c0 += cpp) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    const int c = c0 + tid % cpp;
    if (tid < cpp * rpp && c < W) {
      int r = r0 + tid / cpp;
      for (; r + 3 * rpp < r1; r += 4 * rpp) {        // four independent loads in flight
        a0 += ldf(x + (long long)r * ld + c);
        a1 += ldf(x + (long long)(r + rpp) * ld + c);
        a2 += ldf(x + (long long)(r + 2 * rpp) * ld + c);
        a3 += ldf(x + (long long)(r + 3 * rpp) * ld + c);
      }
      for (; r < r1; r += rpp) a0 += ldf(x + (long long)r * ld + c);
    }
    red[tid] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (tid < cpp && c0 + tid < W) {
      float sum = 0.f;
      for (int qq = 0; qq < rpp; ++qq) sum += red[qq * cpp + tid];
      atomicAdd(&out[c0 + tid], sum);
    }
    __syncthreads();
  }
}

// Vectorised column sums: a thread owns 8 consecutive columns (one 16/32-byte load per row),
// W/8 threads cover a row, 256/(W/8) rows are read concurrently and each thread keeps 4 rows in
// flight; per-block partials are reduced in shared memory, then one atomic per column per block.
__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const bf16* p, float* v) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) { v[2 * i] = sm100::bf16_lo(w[i]); v[2 * i + 1] = sm100::bf16_hi(w[i]); }
}

template <typename T>
__global__ void __launch_bounds__(256) colsum8_kernel(const T* __restrict__ x, int rows, int W, int ld,
                                                      int rows_per_block, float* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[256 * 8];
  const int tpr = W / 8, rpp = 256 / tpr;
  const int tid = threadIdx.x;
  const int cg = tid % tpr, rg = tid / tpr;
  const int r0 = blockIdx.x * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (rg < rpp) {
    int r = r0 + rg;
    for (; r + 3 * rpp < r1; r += 4 * rpp) {
      float v0[8], v1[8], v2[8], v3[8];
      load8(x + (long long)r * ld + cg * 8, v0);
      load8(x + (long long)(r + rpp) * ld + cg * 8, v1);
      load8(x + (long long)(r + 2 * rpp) * ld + cg * 8, v2);
      load8(x + (long long)(r + 3 * rpp) * ld + cg * 8, v3);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += (v0[i] + v1[i]) + (v2[i] + v3[i]);
    }
    for (; r < r1; r += rpp) {
      float v0[8];
      load8(x + (long long)r * ld + cg * 8, v0);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v0[i];
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[tid * 8 + i] = acc[i];     // = red[rg][cg*8+i] (row-group major)
  __syncthreads();
  for (int c = tid; c < W; c += 256) {
    float s = 0.f;
    for (int q = 0; q < rpp; ++q) s += red[q * W + c];
    atomicAdd(&out[c], s);
  }
}

template <typename T>
void colsum_launch(const T* x, int rows, int W, int ld, float* out, cudaStream_t st) {
  if (rows <= 0) return;
  const bool vec = W % 8 == 0 && W <= 2048 && 256 % (W / 8) == 0 && ld % 8 == 0 &&
                   (reinterpret_cast<uintptr_t>(x) % 16) == 0;
  if (vec) {
    const int rpp = 256 / (W / 8);
    const int rpb = std::max(rpp * 8, cdiv(rows, 148 * 8) / rpp * rpp);
    launch(colsum8_kernel<T>, cdiv(rows, rpb), 256, 0, st, x, rows, W, ld, rpb, out);
  } else {
    const int rpb = std::max(64, cdiv(rows, 148 * 2));
    launch(colsum_kernel<T>, cdiv(rows, rpb), 256, 0, st, x, rows, W, ld, rpb, out);
  }
}

void colsum_f32(const float* x, int rows, int W, int ld, float* out, cudaStream_t st) {
  colsum_launch<float>(x, rows, W, ld, out, st);
}
void colsum_bf16(const bf16* x, int rows, int W, int ld, float* out, cudaStream_t st) {
  colsum_launch<bf16>(x, rows, W, ld, out, st);
}

__global__ void cast_rows_kernel(const float* x, int rows, int W, int ldx, bf16* y, int ldy, const float* rowmask) {
  pdl_trigger();
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * W) return;
  const int r = (int)(i / W), c = (int)(i % W);
  float v = x[(long long)r * ldx + c];
  if (rowmask) v *= rowmask[r];
  y[(long long)r * ldy + c] = __float2bfloat16(v);
}
void cast_rows_bf16(const float* x, int rows, int W, int ldx, bf16* y, int ldy, const float* rowmask, cudaStream_t st) {
  const long long n = (long long)rows * W;
  if (n) launch(cast_rows_kernel, cdiv(n, 256), 256, 0, st, x, rows, W, ldx, y, ldy, rowmask);
}

__global__ void mul_rows_kernel(float* x, int rows, int W, const float* rowmask) {
  pdl_trigger();
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * W) return;
  x[i] *= rowmask[i / W];
}
void mul_rows_inplace(float* x, int rows, int W, const float* rowmask, cudaStream_t st) {
  const long long n = (long long)rows * W;
  if (n) launch(mul_rows_kernel, cdiv(n, 256), 256, 0, st, x, rows, W, rowmask);
}

template <int ADD>
__global__ void move_rows_kernel(const float* src, int batch, int src_rows, int src_off, int n, float* dst,
                                 int dst_rows, int dst_off, int W) {
  pdl_trigger();
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)batch * n * W) return;
  const int c = (int)(i % W);
  const long long r = i / W;
  const int b = (int)(r / n), j = (int)(r % n);
  const float v = src[((long long)b * src_rows + src_off + j) * W + c];
  float* d = dst + ((long long)b * dst_rows + dst_off + j) * W + c;
  if (ADD) *d += v; else *d = v;
}
// 16-byte version (W % 4 == 0, 16-byte aligned bases)
template <int ADD>
__global__ void move_rows4_kernel(const float4* src, int batch, int src_rows, int src_off, int n, float4* dst,
                                  int dst_rows, int dst_off, int W4) {
  pdl_trigger();
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)batch * n * W4) return;
  const int c = (int)(i % W4);
  const long long r = i / W4;
  const int b = (int)(r / n), j = (int)(r % n);
  const float4 v = src[((long long)b * src_rows + src_off + j) * W4 + c];
  float4* d = dst + ((long long)b * dst_rows + dst_off + j) * W4 + c;
  if (ADD) {
    float4 o = *d;
    o.x += v.x; o.y += v.y; o.z += v.z; o.w += v.w;
    *d = o;
  } else {
    *d = v;
  }
}
template <int ADD>
static void move_rows(const float* src, int batch, int src_rows, int src_off, int n, float* dst, int dst_rows,
                      int dst_off, int W, cudaStream_t st) {
  const long long tot = (long long)batch * n * W;
  if (!tot) return;
  if (W % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0)
    launch(move_rows4_kernel<ADD>, cdiv(tot / 4, 256), 256, 0, st, reinterpret_cast<const float4*>(src), batch,
           src_rows, src_off, n, reinterpret_cast<float4*>(dst), dst_rows, dst_off, W / 4);
  else
    launch(move_rows_kernel<ADD>, cdiv(tot, 256), 256, 0, st, src, batch, src_rows, src_off, n, dst, dst_rows, dst_off, W);
}
void gather_rows_f32(const float* src, int batch, int src_rows, int src_off, int n, float* dst, int dst_rows,
                     int dst_off, int W, cudaStream_t st) {
  move_rows<0>(src, batch, src_rows, src_off, n, dst, dst_rows, dst_off, W, st);
}
void add_rows_f32(const float* src, int batch, int src_rows, int src_off, int n, float* dst, int dst_rows,
                  int dst_off, int W, cudaStream_t st) {
  move_rows<1>(src, batch, src_rows, src_off, n, dst, dst_rows, dst_off, W, st);
}

// ============================================================== grouped attention (InnerTrans)
// grouped_attention (pkg/src/longrec/tensors.py:406-444): softmax(q kᵀ/√w) v inside each group of
// K consecutive rows.  A CTA stages a tile of whole groups (qkv = [q | k | v] fp32 [T, 3w]) in
// shared memory with coalesced loads, one thread computes one row, and results leave through
// shared memory with coalesced stores.
template <int KT>
__global__ void group_attn_fwd_kernel(const float* __restrict__ qkv, int T, int Kr, int w, bf16* ctx, float* probs) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int K = KT > 0 ? KT : Kr;
  const int TT = (blockDim.x / K) * K;                   // tokens per tile (whole groups)
  const int ld = 3 * w + 1;
  float* s_in = sm;                                      // TT * ld
  float* s_out = sm + TT * ld;                           // TT * (w+1)
  const long long t0 = (long long)blockIdx.x * TT;
  const int nt = (int)min((long long)TT, T - t0);
  for (int e = threadIdx.x; e < nt * 3 * w; e += blockDim.x)
    s_in[(e / (3 * w)) * ld + e % (3 * w)] = qkv[t0 * 3 * w + e];
  __syncthreads();
  const int i = threadIdx.x;
  if (i < nt) {
    const int g0 = i - i % K;
    const float scale = rsqrtf((float)w);
    constexpr int KM = KT > 0 ? KT : 16;
    float s[KM];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (j >= K) break;
      float acc = 0.f;
      for (int c = 0; c < w; ++c) acc = fmaf(s_in[i * ld + c], s_in[(g0 + j) * ld + w + c], acc);
      s[j] = acc * scale;
      mx = fmaxf(mx, s[j]);
    }
    float tot = 0.f;
#pragma unroll
    for (int j = 0; j < KM; ++j) { if (j >= K) break; s[j] = __expf(s[j] - mx); tot += s[j]; }
    const float inv = 1.f / tot;
#pragma unroll
    for (int j = 0; j < KM; ++j) { if (j >= K) break; s[j] *= inv; probs[(t0 + i) * K + j] = s[j]; }
    for (int c = 0; c < w; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < KM; ++j) { if (j >= K) break; acc = fmaf(s[j], s_in[(g0 + j) * ld + 2 * w + c], acc); }
      s_out[i * (w + 1) + c] = acc;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nt * w; e += blockDim.x)
    ctx[t0 * w + e] = __float2bfloat16(s_out[(e / w) * (w + 1) + e % w]);
}

template <int KT>
__global__ void group_attn_bwd_kernel(const float* __restrict__ qkv, const float* __restrict__ probs,
                                      const float* __restrict__ dctx, int T, int Kr, int w, bf16* dqkv) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int K = KT > 0 ? KT : Kr;
  const int TT = (blockDim.x / K) * K;
  const int ld = 3 * w + 1;
  float* s_in = sm;                          // TT * ld   (q|k|v)
  float* s_do = s_in + TT * ld;              // TT * (w+1)
  float* s_out = s_do + TT * (w + 1);        // TT * ld   (dq|dk|dv)
  const long long t0 = (long long)blockIdx.x * TT;
  const int nt = (int)min((long long)TT, T - t0);
  for (int e = threadIdx.x; e < nt * 3 * w; e += blockDim.x)
    s_in[(e / (3 * w)) * ld + e % (3 * w)] = qkv[t0 * 3 * w + e];
  for (int e = threadIdx.x; e < nt * w; e += blockDim.x) s_do[(e / w) * (w + 1) + e % w] = dctx[t0 * w + e];
  __syncthreads();
  const int me_t = threadIdx.x;
  if (me_t < nt) {
    const int g0 = me_t - me_t % K;
    const int me = me_t - g0;
    const float scale = rsqrtf((float)w);
    constexpr int KM = KT > 0 ? KT : 16;
    // dP[i][j] = dctx[i]·v[j];  dS = P ∘ (dP − rowsum(dP∘P)) · scale
    float dS[KM][KM], P[KM][KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) {
      if (i >= K) break;
      float dp[KM];
      float dot = 0.f;
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        if (j >= K) break;
        float acc = 0.f;
        for (int c = 0; c < w; ++c) acc = fmaf(s_do[(g0 + i) * (w + 1) + c], s_in[(g0 + j) * ld + 2 * w + c], acc);
        dp[j] = acc;
        P[i][j] = probs[(t0 + g0 + i) * K + j];
        dot += acc * P[i][j];
      }
#pragma unroll
      for (int j = 0; j < KM; ++j) { if (j >= K) break; dS[i][j] = P[i][j] * (dp[j] - dot) * scale; }
    }
    for (int c = 0; c < w; ++c) {
      float dq = 0.f, dk = 0.f, dv = 0.f;
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        if (j >= K) break;
        dq = fmaf(dS[me][j], s_in[(g0 + j) * ld + w + c], dq);
        dk = fmaf(dS[j][me], s_in[(g0 + j) * ld + c], dk);
        dv = fmaf(P[j][me], s_do[(g0 + j) * (w + 1) + c], dv);
      }
      s_out[me_t * ld + c] = dq;
      s_out[me_t * ld + w + c] = dk;
      s_out[me_t * ld + 2 * w + c] = dv;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nt * 3 * w; e += blockDim.x)
    dqkv[t0 * 3 * w + e] = __float2bfloat16(s_out[(e / (3 * w)) * ld + e % (3 * w)]);
}

void group_attn_fwd(const float* qkv, int T, int K, int w, bf16* ctx, float* probs, cudaStream_t st) {
  const int TT = (128 / K) * K;
  const int smem = 4 * (TT * (3 * w + 1) + TT * (w + 1));
  smem_attr(group_attn_fwd_kernel<2>, 200 * 1024);
  smem_attr(group_attn_fwd_kernel<4>, 200 * 1024);
  smem_attr(group_attn_fwd_kernel<8>, 200 * 1024);
  smem_attr(group_attn_fwd_kernel<0>, 200 * 1024);
  const int grid = cdiv(T, TT);
  if (K == 2) launch(group_attn_fwd_kernel<2>, grid, 128, smem, st, qkv, T, K, w, ctx, probs);
  else if (K == 4) launch(group_attn_fwd_kernel<4>, grid, 128, smem, st, qkv, T, K, w, ctx, probs);
  else if (K == 8) launch(group_attn_fwd_kernel<8>, grid, 128, smem, st, qkv, T, K, w, ctx, probs);
  else launch(group_attn_fwd_kernel<0>, grid, 128, smem, st, qkv, T, K, w, ctx, probs);
}
void group_attn_bwd(const float* qkv, const float* probs, const float* dctx, int T, int K, int w, bf16* dqkv,
                    cudaStream_t st) {
  const int TT = (128 / K) * K;
  const int smem = 4 * (2 * TT * (3 * w + 1) + TT * (w + 1));
  smem_attr(group_attn_bwd_kernel<2>, 220 * 1024);
  smem_attr(group_attn_bwd_kernel<4>, 220 * 1024);
  smem_attr(group_attn_bwd_kernel<8>, 220 * 1024);
  smem_attr(group_attn_bwd_kernel<0>, 220 * 1024);
  const int grid = cdiv(T, TT);
  if (K == 2) launch(group_attn_bwd_kernel<2>, grid, 128, smem, st, qkv, probs, dctx, T, K, w, dqkv);
  else if (K == 4) launch(group_attn_bwd_kernel<4>, grid, 128, smem, st, qkv, probs, dctx, T, K, w, dqkv);
  else if (K == 8) launch(group_attn_bwd_kernel<8>, grid, 128, smem, st, qkv, probs, dctx, T, K, w, dqkv);
  else launch(group_attn_bwd_kernel<0>, grid, 128, smem, st, qkv, probs, dctx, T, K, w, dqkv);
}

// ============================================================== hybrid attention
// _multi_head_attention + masked_softmax (pkg/src/longrec/attention.py:153-169,
// tensors.py:323-351) for one (sample, head) per CTA: Q staged in smem, K/V streamed in chunks,
// one warp per query row with an fp32 online softmax.  Fully-masked rows give ctx = 0.
constexpr int kAttnChunk = 64;

__global__ void attn_fwd_kernel(AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int b = blockIdx.x / a.heads, h = blockIdx.x % a.heads;
  const int dh = a.D / a.heads;
  const int ldp = dh + 1;                                  // padded rows: conflict-free
  float* sQ = sm;                                          // nq * ldp
  float* sK = sQ + a.nq * ldp;                             // chunk * ldp
  float* sV = sK + kAttnChunk * ldp;
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  const float scale = rsqrtf((float)dh);
  const VisRule vis{a.k, a.G, a.ns, a.goff, a.npg[b], a.qg ? a.qg + (long long)b * a.k : nullptr, a.learn,
                     a.self_keys};
  const bf16* Q = a.Q + b * a.sq + h * dh;
  const bf16* Kg = a.Kp + b * a.sk + h * dh;
  const bf16* Vg = a.V + b * a.sv + h * dh;
  for (int i = threadIdx.x; i < a.nq * dh; i += blockDim.x)
    sQ[(i / dh) * ldp + i % dh] = __bfloat162float(Q[(long long)(i / dh) * a.ldq + i % dh]) * scale;
  constexpr int MAXD = 8;                                  // dh <= 256
  const int nd = (dh + 31) / 32;
  const int myq = (a.nq + nw - 1) / nw;                    // queries per warp (<= 8)
  float m_[8], l_[8], acc[8][MAXD];
  for (int r = 0; r < 8; ++r) {
    m_[r] = -INFINITY; l_[r] = 0.f;
    for (int u = 0; u < MAXD; ++u) acc[r][u] = 0.f;
  }
  for (int c0 = 0; c0 < a.nk; c0 += kAttnChunk) {
    const int cn = min(kAttnChunk, a.nk - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * dh; i += blockDim.x) {
      const int r = i / dh, c = i % dh;
      sK[r * ldp + c] = __bfloat162float(Kg[(long long)(c0 + r) * a.ldk + c]);
      sV[r * ldp + c] = __bfloat162float(Vg[(long long)(c0 + r) * a.ldv + c]);
    }
    __syncthreads();
#pragma unroll 1
    for (int r = 0; r < myq && r < 8; ++r) {
      const int i = wid + r * nw;
      if (i >= a.nq) break;
      float s[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int j = lane + 32 * hh;
        float v = -INFINITY;
        if (j < cn && vis(i, c0 + j)) {
          float dot = 0.f;
          for (int c = 0; c < dh; ++c) dot = fmaf(sQ[i * ldp + c], sK[j * ldp + c], dot);
          v = dot;
        }
        s[hh] = v;
      }
      const float cmax = warp_max(fmaxf(s[0], s[1]));
      if (cmax == -INFINITY) continue;                      // nothing visible in this chunk
      const float mnew = fmaxf(m_[r], cmax);
      const float corr = __expf(m_[r] - mnew);
      const float p0 = __expf(s[0] - mnew), p1 = __expf(s[1] - mnew);
      l_[r] = l_[r] * corr + warp_sum(p0 + p1);
      m_[r] = mnew;
      for (int u = 0; u < nd; ++u) acc[r][u] *= corr;
      for (int j = 0; j < cn; ++j) {
        const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31);
        if (pj == 0.f) continue;
        for (int u = 0; u < nd; ++u) {
          const int c = lane + 32 * u;
          if (c < dh) acc[r][u] = fmaf(pj, sV[j * ldp + c], acc[r][u]);
        }
      }
    }
  }
  for (int r = 0; r < myq && r < 8; ++r) {
    const int i = wid + r * nw;
    if (i >= a.nq) break;
    const float inv = l_[r] > 0.f ? 1.f / l_[r] : 0.f;
    bf16* o = a.ctx + b * a.sc + (long long)i * a.ldc + h * dh;
    float* o32 = a.ctx32 + b * a.sc + (long long)i * a.ldc + h * dh;
    for (int u = 0; u < nd; ++u) {
      const int c = lane + 32 * u;
      if (c < dh) {
        o[c] = __float2bfloat16(acc[r][u] * inv);
        o32[c] = acc[r][u] * inv;
      }
    }
    if (lane == 0) a.lse[((long long)b * a.heads + h) * a.nq + i] = l_[r] > 0.f ? m_[r] + __logf(l_[r]) : -INFINITY;
  }
}

void attn_fwd(const AttnArgs& a, cudaStream_t st) {
  const int dh = a.D / a.heads;
  const int smem = 4 * (a.nq + 2 * kAttnChunk) * (dh + 1);
  smem_attr(attn_fwd_kernel, 200 * 1024);
  const int threads = std::min(1024, 32 * std::max(4, (a.nq + 7) / 8));
  launch(attn_fwd_kernel, a.B * a.heads, threads, smem, st, a);
}

// Backward (masked_softmax bw p⊙(g−Σg⊙p), tensors.py:346-349; matmul bws, tensors.py:219-244).
// P is recomputed from the saved log-sum-exp; dQ accumulates in smem across key chunks.
__global__ void attn_bwd_kernel(AttnArgs a, int C) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int b = blockIdx.x / a.heads, h = blockIdx.x % a.heads;
  const int dh = a.D / a.heads;
  const int ldp = dh + 1;
  const int nq = a.nq;
  float* sQ = sm;                          // nq*ldp (pre-scaled)
  float* sdO = sQ + nq * ldp;              // nq*ldp
  float* sdQ = sdO + nq * ldp;             // nq*ldp
  float* sK = sdQ + nq * ldp;              // C*ldp
  float* sV = sK + C * ldp;       // C*ldp
  float* sP = sV + C * ldp;       // nq*C
  float* sdS = sP + nq * C;       // nq*C
  float* sDi = sdS + nq * C;      // nq
  float* sL = sDi + nq;                    // nq
  const float scale = rsqrtf((float)dh);
  const VisRule vis{a.k, a.G, a.ns, a.goff, a.npg[b], a.qg ? a.qg + (long long)b * a.k : nullptr, a.learn,
                     a.self_keys};
  const bf16* Q = a.Q + b * a.sq + h * dh;
  const bf16* Kg = a.Kp + b * a.sk + h * dh;
  const bf16* Vg = a.V + b * a.sv + h * dh;
  const float* dO = a.dctx + b * a.sdc + h * dh;
  const float* O = a.ctx32 + b * a.sc + h * dh;        // fp32 context: D_i consistent with P·V
  for (int i = threadIdx.x; i < nq * dh; i += blockDim.x) {
    const int r = i / dh, c = i % dh;
    sQ[r * ldp + c] = __bfloat162float(Q[(long long)r * a.ldq + c]) * scale;
    sdO[r * ldp + c] = dO[(long long)r * a.lddc + c];
    sdQ[r * ldp + c] = 0.f;
  }
  __syncthreads();
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  for (int i = wid; i < nq; i += nw) {                      // D_i = rowsum(dO ∘ O)
    float s = 0.f;
    for (int c = lane; c < dh; c += 32) s += sdO[i * ldp + c] * O[(long long)i * a.ldc + c];
    s = warp_sum(s);
    if (lane == 0) { sDi[i] = s; sL[i] = a.lse[((long long)b * a.heads + h) * nq + i]; }
  }
  for (int c0 = 0; c0 < a.nk; c0 += C) {
    const int cn = min(C, a.nk - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * dh; i += blockDim.x) {
      const int r = i / dh, c = i % dh;
      sK[r * ldp + c] = __bfloat162float(Kg[(long long)(c0 + r) * a.ldk + c]);
      sV[r * ldp + c] = __bfloat162float(Vg[(long long)(c0 + r) * a.ldv + c]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nq * C; e += blockDim.x) {
      const int i = e / C, j = e % C;
      float p = 0.f, ds = 0.f;
      if (j < cn && sL[i] != -INFINITY && vis(i, c0 + j)) {
        float s = 0.f, dp = 0.f;
        for (int c = 0; c < dh; ++c) {
          s = fmaf(sQ[i * ldp + c], sK[j * ldp + c], s);
          dp = fmaf(sdO[i * ldp + c], sV[j * ldp + c], dp);
        }
        p = __expf(s - sL[i]);
        ds = p * (dp - sDi[i]);
      }
      sP[i * C + j] = p;
      sdS[i * C + j] = ds;
    }
    __syncthreads();
    // dV[j] = Σ_i P[i,j] dO[i];  dK[j] = scale Σ_i dS[i,j] Q̃[i]/scale... (sQ is pre-scaled: Q̃ = scale·Q)
    for (int e = threadIdx.x; e < cn * dh; e += blockDim.x) {
      const int j = e / dh, c = e % dh;
      float dv = 0.f, dk = 0.f;
      for (int i = 0; i < nq; ++i) {
        dv = fmaf(sP[i * C + j], sdO[i * ldp + c], dv);
        dk = fmaf(sdS[i * C + j], sQ[i * ldp + c], dk);
      }
      a.dV[b * a.sdv + (long long)(c0 + j) * a.lddv + h * dh + c] = __float2bfloat16(dv);
      a.dK[b * a.sdk + (long long)(c0 + j) * a.lddk + h * dh + c] = __float2bfloat16(dk);
    }
    for (int e = threadIdx.x; e < nq * dh; e += blockDim.x) {
      const int i = e / dh, c = e % dh;
      float dq = 0.f;
      for (int j = 0; j < cn; ++j) dq = fmaf(sdS[i * C + j], sK[j * ldp + c], dq);
      sdQ[i * ldp + c] += dq * scale;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nq * dh; e += blockDim.x) {
    const int i = e / dh, c = e % dh;
    a.dQ[b * a.sdq + (long long)i * a.lddq + h * dh + c] = __float2bfloat16(sdQ[i * ldp + c]);
  }
}

void attn_bwd(const AttnArgs& a, cudaStream_t st) {
  const int dh = a.D / a.heads;
  const int ldp = dh + 1;
  // key chunk: 64 unless the head width needs a smaller one to fit shared memory (e.g. 256)
  int C = kAttnChunk;
  auto smem_for = [&](int c) { return 4 * (3 * a.nq * ldp + 2 * c * ldp + 2 * a.nq * c + 2 * a.nq); };
  while (C > 8 && smem_for(C) > 220 * 1024) C /= 2;
  const int smem = smem_for(C);
  smem_attr(attn_bwd_kernel, 220 * 1024);
  launch(attn_bwd_kernel, a.B * a.heads, 256, smem, st, a, C);
}

// ============================================================== global tokens
// nontarget_global_tokens / target_global_token raw rows (pkg/src/longrec/inputs.py:500-537),
// before the shared global MLP (which runs as tcgen05 GEMMs).  One CTA per sample.
__global__ void globals_raw_fwd_kernel(GlobalsArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float s_u[64], s_tf[64], s_td[64];
  const int b = blockIdx.x;
  const int F = a.d_item + a.d_act + a.d_time;
  int uid = a.uid[b], cand = a.cand_item[b];
  for (int i = threadIdx.x; i < a.d; i += blockDim.x) s_u[i] = a.uid_tab[(long long)uid * a.d + i];
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    float v = 0.f;
    if (f < a.d_item) v = a.item_tab[(long long)cand * a.d_item + f];
    else if (f >= a.d_item + a.d_act) v = a.time_tab[f - a.d_item - a.d_act];   // time bucket 0
    s_tf[f] = v;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
    float acc = a.tok_b[c];
    for (int f = 0; f < F; ++f) acc = fmaf(s_tf[f], a.tok_w[f * a.d + c], acc);
    s_td[c] = acc;
    a.td[(long long)b * a.d + c] = acc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < a.D; c += blockDim.x) {
    float u = a.lift_b[c], t = a.lift_b[c];
    for (int i = 0; i < a.d; ++i) {
      u = fmaf(s_u[i], a.lift_w[i * a.D + c], u);
      t = fmaf(s_td[i], a.lift_w[i * a.D + c], t);
    }
    const long long r0 = (long long)b * a.m;
    a.raw[(r0) * a.D + c] = u;
    a.raw[(r0 + a.m - 1) * a.D + c] = t;
    a.raw_bf[(r0) * a.D + c] = __float2bfloat16(u);
    a.raw_bf[(r0 + a.m - 1) * a.D + c] = __float2bfloat16(t);
    for (int r = 1; r < a.m - 1; ++r) {
      const float v = a.cls[(r - 1) * a.D + c];
      a.raw[(r0 + r) * a.D + c] = v;
      a.raw_bf[(r0 + r) * a.D + c] = __float2bfloat16(v);
    }
  }
}

__global__ void check_sample_ids_kernel(const int32_t* uid, const int32_t* profile, const int32_t* cand, int B,
                                        int n_users, int n_profiles, int vocab, int32_t* out, int* status) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int u = uid[b], p = profile[b], c = cand ? cand[b] : 0;
  const bool bu = u < 0 || u >= n_users, bp = p < 0 || p >= n_profiles, bc = c < 0 || c >= vocab;
  out[b] = bu ? 0 : u;
  out[B + b] = bp ? 0 : p;
  out[2 * B + b] = bc ? 0 : c;
  if (bu || bp || bc) atomicOr(status, 1);
}

void check_sample_ids(const int32_t* uid, const int32_t* profile, const int32_t* cand, int B, int n_users,
                      int n_profiles, int vocab, int32_t* out, int* status, cudaStream_t st) {
  launch(check_sample_ids_kernel, cdiv(B, 128), 128, 0, st, uid, profile, cand, B, n_users, n_profiles, vocab, out,
         status);
}

void globals_raw_fwd(const GlobalsArgs& a, cudaStream_t st) {
  launch(globals_raw_fwd_kernel, a.B, 128, 0, st, a);
}

// Backward of the raw global rows: lift / token-projection / cls / table gradients, accumulated
// per CTA in shared memory over a slice of samples, then flushed with one atomic per entry.
__global__ void globals_raw_bwd_kernel(GlobalsArgs a, int per_block) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float sm[];
  const int F = a.d_item + a.d_act + a.d_time;
  float* s_lw = sm;                       // d*D
  float* s_lb = s_lw + a.d * a.D;         // D
  float* s_cls = s_lb + a.D;              // (m-2)*D
  float* s_tw = s_cls + (a.m - 2) * a.D;  // F*d
  float* s_tb = s_tw + F * a.d;           // d
  float* s_vec = s_tb + a.d;              // scratch: u[d], td[d], dtd[d], tf[F]
  const int tot = a.d * a.D + a.D + (a.m - 2) * a.D + F * a.d + a.d;
  for (int i = threadIdx.x; i < tot; i += blockDim.x) sm[i] = 0.f;
  float* s_u = s_vec;
  float* s_td = s_u + 64;
  float* s_dtd = s_td + 64;
  float* s_tf = s_dtd + 64;
  __syncthreads();
  const int b0 = blockIdx.x * per_block;
  for (int b = b0; b < min(a.B, b0 + per_block); ++b) {
    const int uid = a.uid[b], cand = a.cand_item[b];
    const float* d0 = a.draw + (long long)b * a.m * a.D;
    const float* dl = d0 + (long long)(a.m - 1) * a.D;
    for (int i = threadIdx.x; i < a.d; i += blockDim.x) {
      s_u[i] = a.uid_tab[(long long)uid * a.d + i];
      s_td[i] = a.td[(long long)b * a.d + i];
    }
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      float v = 0.f;
      if (f < a.d_item) v = a.item_tab[(long long)cand * a.d_item + f];
      else if (f >= a.d_item + a.d_act) v = a.time_tab[f - a.d_item - a.d_act];
      s_tf[f] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < a.d * a.D; e += blockDim.x) {
      const int i = e / a.D, c = e % a.D;
      s_lw[e] += s_u[i] * d0[c] + s_td[i] * dl[c];
    }
    for (int c = threadIdx.x; c < a.D; c += blockDim.x) {
      s_lb[c] += d0[c] + dl[c];
      for (int r = 1; r < a.m - 1; ++r) s_cls[(r - 1) * a.D + c] += d0[(long long)r * a.D + c];
    }
    // d uid_emb and d td (both through lift_w): one warp per dot product of length D
    const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
    for (int i = wid; i < 2 * a.d; i += nw) {
      const int ii = i % a.d;
      const float* src = i < a.d ? d0 : dl;
      float acc = 0.f;
      for (int c = lane; c < a.D; c += 32) acc = fmaf(src[c], a.lift_w[ii * a.D + c], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        if (i < a.d) atomicAdd(&a.g_uid[(long long)uid * a.d + ii], acc);
        else s_dtd[ii] = acc;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < F * a.d; e += blockDim.x) {
      const int f = e / a.d, i = e % a.d;
      s_tw[e] += s_tf[f] * s_dtd[i];
    }
    for (int i = threadIdx.x; i < a.d; i += blockDim.x) s_tb[i] += s_dtd[i];
    for (int f = wid; f < F; f += nw) {                          // one warp per feature row
      if (f >= a.d_item && f < a.d_item + a.d_act) continue;     // zero action slot is a constant
      float acc = 0.f;
      for (int i = lane; i < a.d; i += 32) acc = fmaf(s_dtd[i], a.tok_w[f * a.d + i], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        if (f < a.d_item) atomicAdd(&a.g_item[(long long)cand * a.d_item + f], acc);
        else atomicAdd(&a.g_time[f - a.d_item - a.d_act], acc);
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < a.d * a.D; e += blockDim.x) atomicAdd(&a.g_lift_w[e], s_lw[e]);
  for (int c = threadIdx.x; c < a.D; c += blockDim.x) atomicAdd(&a.g_lift_b[c], s_lb[c]);
  for (int e = threadIdx.x; e < (a.m - 2) * a.D; e += blockDim.x) atomicAdd(&a.g_cls[e], s_cls[e]);
  for (int e = threadIdx.x; e < F * a.d; e += blockDim.x) atomicAdd(&a.g_tok_w[e], s_tw[e]);
  for (int i = threadIdx.x; i < a.d; i += blockDim.x) atomicAdd(&a.g_tok_b[i], s_tb[i]);
}

void globals_raw_bwd(const GlobalsArgs& a, cudaStream_t st) {
  const int F = a.d_item + a.d_act + a.d_time;
  const int smem = 4 * (a.d * a.D + a.D + (a.m - 2) * a.D + F * a.d + a.d + 3 * 64 + 64);
  smem_attr(globals_raw_bwd_kernel, 200 * 1024);
  constexpr int per = 1;   // samples per block: 1 measured best (2: +6 µs, 8: +70 µs)
  launch(globals_raw_bwd_kernel, cdiv(a.B, per), 256, smem, st, a, per);
}

// ============================================================== query selection (model.py:58-123)
// One thread per sample; a bitmap over the merged groups (≤ 8192) realises recent_uniform's set
// with deduplication and newest-first backfill, then emits the picks in group order.
__global__ void select_queries_kernel(const int32_t* npg, int B, int G, int k, int strategy, int32_t* qg) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ uint32_t s_bits[];
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int words = (G + 31) / 32;
  uint32_t* bits = s_bits + threadIdx.x * words;
  if (b >= B) return;
  int32_t* out = qg + (long long)b * k;
  const int fv = min(max(npg[b], 0), G);
  const int nm = G - fv;
  auto cdiv_i = [](long long x, long long y) { return (int)((x + y - 1) / y); };
  if (nm <= k || strategy == 0) {                 // pad fill + all non-pad == the k newest groups
    for (int j = 0; j < k; ++j) out[j] = G - k + j;
    return;
  }
  if (strategy == 1) {                             // uniform
    for (int j = 0; j < k; ++j) out[j] = fv + cdiv_i((long long)(j + 1) * nm, k) - 1;
    return;
  }
  // recent_uniform
  for (int w = 0; w < words; ++w) bits[w] = 0u;
  const int r = (k + 1) / 2, u = k - r;
  int cnt = 0;
  auto pick = [&](int g) {
    const uint32_t m = 1u << (g & 31);
    if (!(bits[g >> 5] & m)) { bits[g >> 5] |= m; ++cnt; }
  };
  for (int g = G - r; g < G; ++g) pick(g);
  const int plen = nm - r;
  for (int j = 0; j < u; ++j) pick(fv + cdiv_i((long long)(j + 1) * plen, u) - 1);
  for (int g = G - 1; g >= fv && cnt < k; --g) pick(g);
  int o = 0;
  for (int g = fv; g < G && o < k; ++g)
    if (bits[g >> 5] & (1u << (g & 31))) out[o++] = g;
}

void select_queries(const int32_t* npg, int B, int G, int k, int strategy, int32_t* qg, cudaStream_t st) {
  const int words = (G + 31) / 32;
  const int per = std::max(1, std::min(64, (48 * 1024) / (words * 4)));
  launch(select_queries_kernel, cdiv(B, per), per, (size_t)per * words * 4, st, npg, B, G, k, strategy, qg);
}

__global__ void gather_query_rows_kernel(const float* merged, const int32_t* qg, const float* bank, int B, int G,
                                         int k, int W, float* O, int q) {
  pdl_trigger();
  pdl_wait();
  const long long n = (long long)B * k * W;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % W);
    const long long bi = e / W;
    const int i = (int)(bi % k), b = (int)(bi / k);
    const float v = bank ? bank[(long long)i * W + c] : merged[((long long)b * G + qg[bi]) * W + c];
    O[((long long)b * q + i) * W + c] = v;
  }
}

void gather_query_rows(const float* merged, const int32_t* qg, const float* bank, int B, int G, int k, int W,
                       float* O, int q, cudaStream_t st) {
  const long long n = (long long)B * k * W;
  if (n) launch(gather_query_rows_kernel, std::min(cdiv(n, 256), 148 * 16), 256, 0, st, merged, qg, bank, B, G, k, W, O, q);
}

__global__ void scatter_query_rows_kernel(const float* dO, int q, const int32_t* qg, int B, int G, int k, int W,
                                          float* dmerged, float* g_bank) {
  pdl_trigger();
  pdl_wait();
  if (g_bank) {                                    // Σ over samples, one thread per (i, c)
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= k * W) return;
    const int i = e / W, c = e % W;
    float acc = 0.f;
    for (int b = 0; b < B; ++b) acc += dO[((long long)b * q + i) * W + c];
    g_bank[e] += acc;
    return;
  }
  const long long n = (long long)B * k * W;        // query groups of one sample are distinct
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % W);
    const long long bi = e / W;
    const int i = (int)(bi % k), b = (int)(bi / k);
    dmerged[((long long)b * G + qg[bi]) * W + c] += dO[((long long)b * q + i) * W + c];
  }
}

void scatter_query_rows(const float* dO, int q, const int32_t* qg, int B, int G, int k, int W, float* dmerged,
                        float* g_bank, cudaStream_t st) {
  if (g_bank) {
    launch(scatter_query_rows_kernel, cdiv((long long)k * W, 256), 256, 0, st, dO, q, qg, B, G, k, W, dmerged, g_bank);
  } else {
    const long long n = (long long)B * k * W;
    if (n) launch(scatter_query_rows_kernel, std::min(cdiv(n, 256), 148 * 16), 256, 0, st, dO, q, qg, B, G, k, W,
                  dmerged, g_bank);
  }
}

// ============================================================== head + BCE
// Head of forward_tensor (pkg/src/longrec/model.py:346-362): [t, c, t⊙c, t⊙t, u_d] → GELU MLP →
// sigmoid; BCE with the 1e-12 clamp (tensors.py:551-571).  One warp per sample: lanes own hidden
// units (coalesced W1 rows, the input row broadcast from shared memory).
constexpr int kHeadWarps = 4;

// W1 [HIN, hh] staged in shared memory with row stride hh+1: conflict-free both for lanes over
// hidden units (forward) and lanes over inputs (backward).
__device__ __forceinline__ void stage_w1(const float* __restrict__ w1, int HIN, int hh, float* s_w) {
  const int n = HIN * hh;
  if ((reinterpret_cast<uintptr_t>(w1) & 15) == 0 && (hh & 3) == 0) {
    // 16-byte loads, eight in flight per thread before their (scalar, padded-stride) stores
    const int n4 = n / 4;
    for (int e0 = threadIdx.x; e0 < n4; e0 += 8 * blockDim.x) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < n4) v[u] = __ldg(reinterpret_cast<const float4*>(w1) + e);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < n4) {
          const int i = (4 * e) / hh, j = (4 * e) % hh;
          float* d = s_w + i * (hh + 1) + j;
          d[0] = v[u].x; d[1] = v[u].y; d[2] = v[u].z; d[3] = v[u].w;
        }
      }
    }
  } else {
#pragma unroll 8
    for (int e = threadIdx.x; e < n; e += blockDim.x) s_w[(e / hh) * (hh + 1) + e % hh] = __ldg(w1 + e);
  }
  __syncthreads();
}

__device__ __forceinline__ void head_row(const float* x, int b, int q, int k, int m, int D, int d, const int32_t* uid,
                                         const int32_t* profile, const float* uid_tab, const float* prof_tab,
                                         float* s_in, int lane) {
  const float* t = x + ((long long)b * q + k + m - 1) * D;
  const float* c = x + ((long long)b * q + k + 1) * D;
  for (int i = lane; i < D; i += 32) {
    const float tv = t[i], cv = c[i];
    s_in[i] = tv; s_in[D + i] = cv; s_in[2 * D + i] = tv * cv; s_in[3 * D + i] = tv * tv;
  }
  const int u = uid[b], pr = profile[b];
  for (int i = lane; i < d; i += 32) {
    s_in[4 * D + i] = uid_tab[(long long)u * d + i];
    s_in[4 * D + d + i] = prof_tab[(long long)pr * d + i];
  }
  __syncwarp();
}

template <bool STAGE>
__global__ void head_fwd_kernel(HeadArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float smem_h[];
  const int D = a.D, HIN = 4 * D + 2 * a.d;
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int ws = STAGE ? a.hh + 1 : a.hh;
  const float* W1 = a.w1;
  float* s_base = smem_h;
  if constexpr (STAGE) {
    stage_w1(a.w1, HIN, a.hh, smem_h);
    W1 = smem_h;
    s_base = smem_h + HIN * ws;
  }
  const int b = blockIdx.x * kHeadWarps + wid;
  if (b >= a.B) return;
  float* s_in = s_base + wid * HIN;
  head_row(a.x, b, a.q, a.k, a.m, D, a.d, a.uid, a.profile, a.uid_tab, a.prof_tab, s_in, lane);
  for (int i = lane; i < HIN; i += 32) a.hin[(long long)b * HIN + i] = s_in[i];
  float zpart = 0.f;
  for (int j = lane; j < a.hh; j += 32) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int i = 0;
    for (; i + 3 < HIN; i += 4) {
      a0 = fmaf(s_in[i], W1[i * ws + j], a0);
      a1 = fmaf(s_in[i + 1], W1[(i + 1) * ws + j], a1);
      a2 = fmaf(s_in[i + 2], W1[(i + 2) * ws + j], a2);
      a3 = fmaf(s_in[i + 3], W1[(i + 3) * ws + j], a3);
    }
    for (; i < HIN; ++i) a0 = fmaf(s_in[i], W1[i * ws + j], a0);
    const float z1 = (a0 + a1) + (a2 + a3) + a.b1[j];
    a.z1[(long long)b * a.hh + j] = z1;
    zpart = fmaf(gelu_f(z1), a.w2[j], zpart);
  }
  const float acc = warp_sum(zpart);
  if (lane == 0) {
    const float z = acc + a.b2[0];
    const float e = __expf(-fabsf(z));
    const float p = z >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
    a.probs[b] = p;
    if (a.loss_per) {
      // bce with the reference's clamp p_c = clip(p, 1e-12, 1-1e-12) (tensors.py:551-571),
      // evaluated in log-odds space: 1 - 1e-12 is not representable in fp32, but
      // log p = -softplus(-z) and log(1-p) = -softplus(z) are, and clamping p at 1e-12 is
      // clamping the log at log(1e-12); the clamp's zero-gradient region is |z| ≥ logit(1-1e-12).
      const float y = a.label[b];
      const float kLog12 = -27.631021115928547f;          // log(1e-12)
      const float sp_pos = fmaxf(z, 0.f) + log1pf(__expf(-fabsf(z)));    // softplus(z)
      const float sp_neg = sp_pos - z;                                   // softplus(-z)
      const float log_p = fmaxf(-sp_neg, kLog12), log_q = fmaxf(-sp_pos, kLog12);
      // a NaN logit must reach the loss (NumericalError, model.py:563-566): fmaxf drops NaN
      a.loss_per[b] = !isnan(z) ? -(y * log_p + (1.f - y) * log_q) : __int_as_float(0x7fc00000);
      const bool inr = fabsf(z) < 27.631021115928547f;
      a.dz[b] = inr ? (p - y) / (float)a.B : 0.f;
    }
  }
}

__global__ void loss_mean_kernel(const float* loss_per, int B, float* loss) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[256];
  float s = 0.f;
  for (int i = threadIdx.x; i < B; i += blockDim.x) s += loss_per[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[0] = red[0] / (float)B;
}

namespace {
int head_smem_w1(const HeadArgs& a) { return 4 * (4 * a.D + 2 * a.d) * (a.hh + 1); }
constexpr int kHeadSmemMax = 200 * 1024;
}  // namespace

void loss_mean(const float* loss_per, int B, float* loss, cudaStream_t st) {
  launch(loss_mean_kernel, 1, 256, 0, st, loss_per, B, loss);
}

void head_fwd(const HeadArgs& a, int with_loss, cudaStream_t st) {
  const int smem = 4 * kHeadWarps * (4 * a.D + 2 * a.d);
  const bool stage = smem + head_smem_w1(a) <= kHeadSmemMax;
  if (stage) {
    smem_attr(head_fwd_kernel<true>, kHeadSmemMax);
    launch(head_fwd_kernel<true>, cdiv(a.B, kHeadWarps), 32 * kHeadWarps, smem + head_smem_w1(a), st, a);
  } else {
    launch(head_fwd_kernel<false>, cdiv(a.B, kHeadWarps), 32 * kHeadWarps, smem, st, a);
  }
  if (with_loss) loss_mean(a.loss_per, a.B, a.loss, st);
}

// Head backward, one warp per sample: dz1 = dz·w2⊙GELU'(z1) (lanes = hidden units), then
// dhin = W1·dz1 with lanes over the inputs, W1 rows read as float4 runs.
template <bool STAGE>
__global__ void head_bwd_kernel(HeadArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float smem_h[];
  const int D = a.D, HIN = 4 * D + 2 * a.d;
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31;
  float* s_base = smem_h;
  if constexpr (STAGE) {
    stage_w1(a.w1, HIN, a.hh, smem_h);
    s_base = smem_h + HIN * (a.hh + 1);
  }
  const int b = blockIdx.x * kHeadWarps + wid;
  if (b >= a.B) return;
  float* s_dz1 = s_base + wid * (a.hh + HIN);
  float* s_dhin = s_dz1 + a.hh;
  const float dz = a.dz[b];
  for (int j = lane; j < a.hh; j += 32) {
    const float v = dz * a.w2[j] * gelu_grad_f(a.z1[(long long)b * a.hh + j]);
    s_dz1[j] = v;
    a.dz1[(long long)b * a.hh + j] = v;
  }
  __syncwarp();
  const bool vec = !STAGE && (a.hh % 4) == 0 && (reinterpret_cast<uintptr_t>(a.w1) & 15) == 0;
  for (int i = lane; i < HIN; i += 32) {
    const float* wr = STAGE ? smem_h + i * (a.hh + 1) : a.w1 + (long long)i * a.hh;
    float acc = 0.f;
    if (vec) {
      for (int j = 0; j < a.hh; j += 4) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(wr + j));
        acc = fmaf(s_dz1[j], w.x, acc); acc = fmaf(s_dz1[j + 1], w.y, acc);
        acc = fmaf(s_dz1[j + 2], w.z, acc); acc = fmaf(s_dz1[j + 3], w.w, acc);
      }
    } else {
      for (int j = 0; j < a.hh; ++j) acc = fmaf(s_dz1[j], wr[j], acc);
    }
    s_dhin[i] = acc;
  }
  __syncwarp();
  const float* hin = a.hin + (long long)b * HIN;
  float* dt = a.dx + ((long long)b * a.q + a.k + a.m - 1) * D;
  float* dc = a.dx + ((long long)b * a.q + a.k + 1) * D;
  bf16* dtb = a.dx_bf ? a.dx_bf + ((long long)b * a.q + a.k + a.m - 1) * D : nullptr;
  bf16* dcb = a.dx_bf ? a.dx_bf + ((long long)b * a.q + a.k + 1) * D : nullptr;
  for (int i = lane; i < D; i += 32) {
    const float t = hin[i], c = hin[D + i];
    const float vt = s_dhin[i] + s_dhin[2 * D + i] * c + 2.f * s_dhin[3 * D + i] * t;
    const float vc = s_dhin[D + i] + s_dhin[2 * D + i] * t;
    dt[i] = vt;
    dc[i] = vc;
    if (dtb) { dtb[i] = __float2bfloat16(vt); dcb[i] = __float2bfloat16(vc); }
  }
  const int uid = a.uid[b], prof = a.profile[b];
  for (int i = lane; i < a.d; i += 32) {
    atomicAdd(&a.g_uid[(long long)uid * a.d + i], s_dhin[4 * D + i]);
    atomicAdd(&a.g_prof[(long long)prof * a.d + i], s_dhin[4 * D + a.d + i]);
  }
}

// head weight gradients: deterministic reductions over the batch (one thread per weight)
// head weight gradients: batch reductions split over gridDim.y sample slices (atomic combine)
__global__ void head_wgrad_kernel(HeadArgs a, int per) {
  pdl_trigger();
  pdl_wait();
  const int HIN = 4 * a.D + 2 * a.d;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_w1 = HIN * a.hh;
  const int b0 = blockIdx.y * per, b1 = min(a.B, b0 + per);
  if (e < n_w1) {
    const int i = e / a.hh, j = e % a.hh;
    float acc0 = 0.f, acc1 = 0.f;
    int b = b0;
    for (; b + 1 < b1; b += 2) {
      acc0 = fmaf(a.hin[(long long)b * HIN + i], a.dz1[(long long)b * a.hh + j], acc0);
      acc1 = fmaf(a.hin[(long long)(b + 1) * HIN + i], a.dz1[(long long)(b + 1) * a.hh + j], acc1);
    }
    if (b < b1) acc0 = fmaf(a.hin[(long long)b * HIN + i], a.dz1[(long long)b * a.hh + j], acc0);
    atomicAdd(&a.g_w1[e], acc0 + acc1);
  } else if (e < n_w1 + a.hh) {
    const int j = e - n_w1;
    float acc = 0.f, acc2 = 0.f;
    for (int b = b0; b < b1; ++b) {
      acc += a.dz1[(long long)b * a.hh + j];
      acc2 = fmaf(gelu_f(a.z1[(long long)b * a.hh + j]), a.dz[b], acc2);
    }
    atomicAdd(&a.g_b1[j], acc);
    atomicAdd(&a.g_w2[j], acc2);
  } else if (e == n_w1 + a.hh) {
    float acc = 0.f;
    for (int b = b0; b < b1; ++b) acc += a.dz[b];
    atomicAdd(&a.g_b2[0], acc);
  }
}

void head_bwd(const HeadArgs& a, cudaStream_t st) {
  const int HIN = 4 * a.D + 2 * a.d;
  const int smem = 4 * kHeadWarps * (a.hh + HIN);
  if (smem + head_smem_w1(a) <= kHeadSmemMax) {
    smem_attr(head_bwd_kernel<true>, kHeadSmemMax);
    launch(head_bwd_kernel<true>, cdiv(a.B, kHeadWarps), 32 * kHeadWarps, smem + head_smem_w1(a), st, a);
  } else {
    launch(head_bwd_kernel<false>, cdiv(a.B, kHeadWarps), 32 * kHeadWarps, smem, st, a);
  }
}

void head_wgrad(const HeadArgs& a, cudaStream_t st) {
  const int HIN = 4 * a.D + 2 * a.d;
  const int n = HIN * a.hh + a.hh + 1;
  const int per = 16;
  launch(head_wgrad_kernel, dim3(cdiv(n, 128), cdiv(a.B, per)), 128, 0, st, a, per);
}

__global__ void dz_from_dprobs_kernel(const float* probs, const float* dprobs, int B, float* dz) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    const float pb = probs[b];
    dz[b] = dprobs[b] * pb * (1.f - pb);
  }
}

void dz_from_dprobs(const float* probs, const float* dprobs, int B, float* dz, cudaStream_t st) {
  launch(dz_from_dprobs_kernel, cdiv(B, 256), 256, 0, st, probs, dprobs, B, dz);
}

// ============================================================== parameters
__global__ void pack_kernel(const float* __restrict__ params, const PackList specs, void* dst) {
  pdl_trigger();
  pdl_wait();
  const CopySpec s = specs.s[blockIdx.y];
  const long long n = (long long)s.rows * s.cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / s.cols), c = (int)(e % s.cols);
    const float v = params[s.src_off + (long long)r * s.src_ld + c];
    const long long o = s.dst_off + (long long)r * s.dst_ld + c;
    if (s.to_bf16) reinterpret_cast<bf16*>(dst)[o] = __float2bfloat16(v);
    else reinterpret_cast<float*>(dst)[o] = v;
  }
}

void pack_params(const float* params, const PackList& specs, void* dst_base, cudaStream_t st) {
  if (specs.n) launch(pack_kernel, dim3(64, specs.n), 256, 0, st, params, specs, dst_base);
}

// Adam (pkg/src/longrec/model.py:467-482)
__global__ void adam_kernel(float* p, const float* g, float* m, float* v, long long n, float lr, float c1, float c2) {
  pdl_trigger();
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = 0.9f * m[i] + 0.1f * gi;
    const float vi = 0.999f * v[i] + 0.001f * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + 1e-8f);
  }
}

// same per-element arithmetic, four elements per 16-byte access (aligned buffers, n % 4 == 0)
__global__ void adam4_kernel(float4* p, const float4* g, float4* m, float4* v, long long n4, float lr, float c1,
                             float c2) {
  pdl_trigger();
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 g4 = g[i];
    float4 m4 = m[i], v4 = v[i], p4 = p[i];
    float* pm = &m4.x; float* pv = &v4.x; float* pp = &p4.x;
    const float* pg = &g4.x;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float gi = pg[u];
      const float mi = 0.9f * pm[u] + 0.1f * gi;
      const float vi = 0.999f * pv[u] + 0.001f * gi * gi;
      pm[u] = mi;
      pv[u] = vi;
      pp[u] -= lr * (mi / c1) / (sqrtf(vi / c2) + 1e-8f);
    }
    m[i] = m4; v[i] = v4; p[i] = p4;
  }
}

void adam_step(float* p, const float* g, float* m, float* v, long long n, float lr, int t, cudaStream_t st) {
  const float c1 = (float)(1.0 - pow(0.9, t)), c2 = (float)(1.0 - pow(0.999, t));
  const bool vec = n % 4 == 0 && ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                                   reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  if (vec)
    launch(adam4_kernel, 148 * 4, 256, 0, st, reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
           reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n / 4, lr, c1, c2);
  else
    launch(adam_kernel, 148 * 8, 256, 0, st, p, g, m, v, n, lr, c1, c2);
}


// ============================================================== head rows of the last block
// The head reads only rows k+1 (CLS) and k+m−1 (target) of the last block's output
// (pkg/src/longrec/model.py:346-362), so that block's row-wise tail runs on those two rows per
// sample: compact row 2b + 0 ↔ full row b·q + k+1, compact row 2b + 1 ↔ full row b·q + k+m−1.
template <typename T, bool GATHER>
__global__ void head_rows_kernel(const T* __restrict__ src, T* __restrict__ dst, int B, int q, int r0, int r1,
                                 int W) {
  pdl_trigger();
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)2 * B * W) return;
  const int c = (int)(i % W), r = (int)(i / W);
  const long long full = (long long)(r >> 1) * q + ((r & 1) ? r1 : r0);
  if (GATHER) dst[(long long)r * W + c] = src[full * W + c];
  else dst[full * W + c] = src[(long long)r * W + c];
}

// gathers move 16-byte vectors when the row width allows (W·sizeof(T) % 16 == 0, aligned bases)
void head_rows_gather_f32(const float* full, float* compact, int B, int q, int r0, int r1, int W, cudaStream_t st) {
  if (W % 4 == 0 && (reinterpret_cast<uintptr_t>(full) & 15) == 0 && (reinterpret_cast<uintptr_t>(compact) & 15) == 0)
    launch(head_rows_kernel<uint4, true>, cdiv((long long)2 * B * W / 4, 256), 256, 0, st,
           reinterpret_cast<const uint4*>(full), reinterpret_cast<uint4*>(compact), B, q, r0, r1, W / 4);
  else
    launch(head_rows_kernel<float, true>, cdiv((long long)2 * B * W, 256), 256, 0, st, full, compact, B, q, r0, r1, W);
}
void head_rows_gather_bf16(const bf16* full, bf16* compact, int B, int q, int r0, int r1, int W, cudaStream_t st) {
  if (W % 8 == 0 && (reinterpret_cast<uintptr_t>(full) & 15) == 0 && (reinterpret_cast<uintptr_t>(compact) & 15) == 0)
    launch(head_rows_kernel<uint4, true>, cdiv((long long)2 * B * W / 8, 256), 256, 0, st,
           reinterpret_cast<const uint4*>(full), reinterpret_cast<uint4*>(compact), B, q, r0, r1, W / 8);
  else
    launch(head_rows_kernel<bf16, true>, cdiv((long long)2 * B * W, 256), 256, 0, st, full, compact, B, q, r0, r1, W);
}
// full[B·q, W] = the compact rows at their places, zero elsewhere (one pass, no separate memset)
__global__ void head_rows_expand_kernel(const float* __restrict__ compact, float* __restrict__ full, int B, int q,
                                        int r0, int r1, int W) {
  pdl_trigger();
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)B * q * W / 4) return;
  const long long e = i * 4;
  const int c = (int)(e % W);
  const long long row = e / W;
  const int b = (int)(row / q), j = (int)(row % q);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j == r0 || j == r1)
    v = *reinterpret_cast<const float4*>(compact + ((long long)2 * b + (j == r1 ? 1 : 0)) * W + c);
  *reinterpret_cast<float4*>(full + e) = v;
}

// both gathers of the compact last-block tail in one launch: bf16 rows (W_b wide) and fp32 rows (W_f
// wide), 16-byte vectors; the first 2B·W_b/8 threads take the bf16 part
__global__ void head_rows_gather2_kernel(const uint4* __restrict__ fb, uint4* __restrict__ cb, int vb,
                                         const uint4* __restrict__ ff, uint4* __restrict__ cf, int vf, int B, int q,
                                         int r0, int r1) {
  pdl_trigger();
  pdl_wait();
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nb = (long long)2 * B * vb;
  const uint4* src = fb;
  uint4* dst = cb;
  int V = vb;
  if (i >= nb) { i -= nb; src = ff; dst = cf; V = vf; }
  if (i >= (long long)2 * B * V) return;
  const int c = (int)(i % V), r = (int)(i / V);
  const long long full = (long long)(r >> 1) * q + ((r & 1) ? r1 : r0);
  dst[(long long)r * V + c] = src[full * V + c];
}

void head_rows_gather_pair(const bf16* full_b, bf16* compact_b, const float* full_f, float* compact_f, int B, int q,
                           int r0, int r1, int W, cudaStream_t st) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (W % 8 == 0 && al(full_b) && al(compact_b) && al(full_f) && al(compact_f)) {
    const long long n = (long long)2 * B * (W / 8 + W / 4);
    launch(head_rows_gather2_kernel, cdiv(n, 256), 256, 0, st, reinterpret_cast<const uint4*>(full_b),
           reinterpret_cast<uint4*>(compact_b), W / 8, reinterpret_cast<const uint4*>(full_f),
           reinterpret_cast<uint4*>(compact_f), W / 4, B, q, r0, r1);
  } else {
    head_rows_gather_bf16(full_b, compact_b, B, q, r0, r1, W, st);
    head_rows_gather_f32(full_f, compact_f, B, q, r0, r1, W, st);
  }
}

// both expansions of the compact tail's gradients in one launch (blockIdx.y picks the pair)
__global__ void head_rows_expand2_kernel(const float* __restrict__ c0, float* __restrict__ f0,
                                         const float* __restrict__ c1, float* __restrict__ f1, int B, int q, int r0,
                                         int r1, int W) {
  pdl_trigger();
  pdl_wait();
  const float* compact = blockIdx.y ? c1 : c0;
  float* full = blockIdx.y ? f1 : f0;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)B * q * W / 4) return;
  const long long e = i * 4;
  const int c = (int)(e % W);
  const long long row = e / W;
  const int b = (int)(row / q), j = (int)(row % q);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j == r0 || j == r1)
    v = *reinterpret_cast<const float4*>(compact + ((long long)2 * b + (j == r1 ? 1 : 0)) * W + c);
  *reinterpret_cast<float4*>(full + e) = v;
}

void head_rows_scatter_pair(const float* c0, float* f0, const float* c1, float* f1, int B, int q, int r0, int r1,
                            int W, cudaStream_t st) {
  if (W % 4 == 0) {
    launch(head_rows_expand2_kernel, dim3((unsigned)cdiv((long long)B * q * W / 4, 256), 2), 256, 0, st, c0, f0, c1,
           f1, B, q, r0, r1, W);
  } else {
    head_rows_scatter_f32(c0, f0, B, q, r0, r1, W, st);
    head_rows_scatter_f32(c1, f1, B, q, r0, r1, W, st);
  }
}

void head_rows_scatter_f32(const float* compact, float* full, int B, int q, int r0, int r1, int W, cudaStream_t st) {
  if (W % 4 == 0) {
    launch(head_rows_expand_kernel, cdiv((long long)B * q * W / 4, 256), 256, 0, st, compact, full, B, q, r0, r1, W);
  } else {
    cudaMemsetAsync(full, 0, (size_t)B * q * W * 4, st);
    launch(head_rows_kernel<float, false>, cdiv((long long)2 * B * W, 256), 256, 0, st, compact, full, B, q, r0, r1, W);
  }
}

}  // namespace longer
