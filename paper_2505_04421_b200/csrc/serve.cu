// serve.cu — KV-cache serving kernels (build_cache / score_with_cache, pkg/src/longrec/serving.py:84-167).
//
// Stage 1 (cache build) runs the ordinary forward for a batch of users with a placeholder candidate
// and keeps every candidate-independent row: the visibility rule (pkg/src/longrec/attention.py:49-87)
// forbids every non-target row from seeing the target, so those rows are exactly the full
// forward's.  Stage 2 pushes only the candidates' target rows — thousands per call, batched over
// users × candidates — through the blocks against the cached keys/values, each with its own k/v
// appended last (attention_block_cached, attention.py:215-236).
#include "fe_common.cuh"
#include "serve.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace longer {

using namespace fe;

namespace {
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
}

// ------------------------------------------------------------------ row copies
__global__ void copy_rows_bf16_kernel(const bf16* src, long long s_stride, int s_ld, int s_col, bf16* dst,
                                      long long d_stride, int rows, int cols, int batch) {
  pdl_trigger();
  pdl_wait();
  const long long n = (long long)batch * rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % cols);
    const long long rr = e / cols;
    const int r = (int)(rr % rows), u = (int)(rr / rows);
    dst[u * d_stride + (long long)r * cols + c] = src[u * s_stride + (long long)r * s_ld + s_col + c];
  }
}

void copy_rows_bf16(const bf16* src, long long s_stride, int s_ld, int s_col, bf16* dst, long long d_stride, int rows,
                    int cols, int batch, cudaStream_t st) {
  const long long n = (long long)batch * rows * cols;
  if (n) launch(copy_rows_bf16_kernel, std::min(cdiv(n, 256), 148 * 16), 256, 0, st, src, s_stride, s_ld, s_col, dst,
                                                                                   d_stride, rows, cols, batch);
}

// per user: CLS output of the last layer, user-side head features [uid_emb | profile_emb], npg
__global__ void cache_user_kernel(CacheUserArgs a) {
  pdl_trigger();
  pdl_wait();
  const int u = blockIdx.x;
  const float* cls = a.x_last + ((long long)u * a.q + a.k + 1) * a.D;
  for (int c = threadIdx.x; c < a.D; c += blockDim.x) a.cls[(long long)u * a.D + c] = cls[c];
  const int uid = a.uid[u], prof = a.profile[u];
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
    a.ud[(long long)u * 2 * a.d + c] = a.uid_tab[(long long)uid * a.d + c];
    a.ud[(long long)u * 2 * a.d + a.d + c] = a.prof_tab[(long long)prof * a.d + c];
  }
  if (threadIdx.x == 0) a.npg_out[u] = a.npg[u];
}

void cache_users(const CacheUserArgs& a, cudaStream_t st) { launch(cache_user_kernel, a.U, 128, 0, st, a); }

// ------------------------------------------------------------------ target rows
// target_global_token (pkg/src/longrec/inputs.py:500-512) before the global MLP:
// [item_emb | 0_act | time_emb[0]] · W_tp + b_tp → · lift_w + lift_b, one CTA per candidate row.
__global__ void target_rows_kernel(TargetArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float s_tf[64], s_td[64];
  const long long r = blockIdx.x;
  const int F = a.d_item + a.d_act + a.d_time;
  int item = a.cand ? a.cand[r] : (int)r;
  if (item < 0 || item >= a.vocab) { if (threadIdx.x == 0) atomicOr(a.status, 1); item = 0; }
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    float v = 0.f;
    if (f < a.d_item) v = a.item_tab[(long long)item * a.d_item + f];
    else if (f >= a.d_item + a.d_act) v = a.time_tab[f - a.d_item - a.d_act];
    s_tf[f] = v;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < a.d; c += blockDim.x) {
    float acc = a.tok_b[c];
    for (int f = 0; f < F; ++f) acc = fmaf(s_tf[f], a.tok_w[f * a.d + c], acc);
    s_td[c] = acc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < a.D; c += blockDim.x) {
    float t = a.lift_b[c];
    for (int i = 0; i < a.d; ++i) t = fmaf(s_td[i], a.lift_w[i * a.D + c], t);
    a.raw_bf[r * a.D + c] = __float2bfloat16(t);
  }
}

void target_rows(const TargetArgs& a, cudaStream_t st) {
  if (a.R) launch(target_rows_kernel, (unsigned)a.R, 128, 0, st, a);
}

// one warp per candidate row: D fp32 (x) + 3D bf16 (q | k_own | v_own) as 16-byte vectors
__global__ void gather_item_rows_kernel(const int32_t* cand, long long R, int vocab, const float* item_x,
                                        const bf16* item_qkv, int D, float* x, bf16* qkv, int* status) {
  pdl_trigger();
  pdl_wait();
  const long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  int item = cand[r];
  if (item < 0 || item >= vocab) { if (lane == 0) atomicOr(status, 1); item = 0; }
  const float4* sx = reinterpret_cast<const float4*>(item_x + (long long)item * D);
  float4* dx = reinterpret_cast<float4*>(x + r * D);
  for (int i = lane; i < D / 4; i += 32) dx[i] = sx[i];
  const uint4* sq = reinterpret_cast<const uint4*>(item_qkv + (long long)item * 3 * D);
  uint4* dq = reinterpret_cast<uint4*>(qkv + r * 3 * D);
  for (int i = lane; i < 3 * D / 8; i += 32) dq[i] = sq[i];
}

void gather_item_rows(const int32_t* cand, long long R, int vocab, const float* item_x, const bf16* item_qkv, int D,
                      float* x, bf16* qkv, int* status, cudaStream_t st) {
  if (R) launch(gather_item_rows_kernel, (unsigned)((R + 7) / 8), 256, 0, st, cand, R, vocab, item_x, item_qkv, D, x, qkv,
                status);
}

// ------------------------------------------------------------------ cached attention
// One CTA per (user, 128-candidate tile, head); two CTAs per SM.  All queries are target rows
// (global rank m-1): they see every non-pad sequence key and every cached global, plus their own
// key appended last (attention_block_cached, attention.py:215-236).  One pass over the cached
// keys: per 128-key chunk, S = Q·Kᵀ on the tensor core (TMEM), the row max / sum online, P (bf16)
// written over the chunk's K tile, O += P·V in TMEM.  The running max m is only moved when a chunk
// exceeds it by more than kRescale (then O is rescaled in TMEM): numerator and denominator share
// the same m, so the result is exact, and P ≤ e^kRescale stays well inside bf16 / fp32 range.  The
// own key is handled in registers.  Rows move between HBM and the canonical tiles with
// warp-cooperative loads (8 rows × 64 contiguous bytes per instruction; conflict-free 16-byte
// shared stores), each worker warp owning the 32 rows of its TMEM lane quarter.
constexpr float kRescale = 8.f;

// the warp's 32 rows [0, 32) of a row-major bf16 matrix (row stride ld) → canonical tile rows
// [t0, t0 + 32) (K = DH); rows ≥ nvalid are zero-filled
template <int DH>
__device__ __forceinline__ void warp_rows_to_canon(bf16* tile, int t0, const bf16* src, long long ld, int nvalid,
                                                   int lane) {
  const int lr = lane & 7, kc = lane >> 3;
  uint4 v[4][DH / 32];
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int k = 0; k < DH / 32; ++k) {
      const int r = rb * 8 + lr;
      v[rb][k] = r < nvalid ? *reinterpret_cast<const uint4*>(src + r * ld + (4 * k + kc) * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int k = 0; k < DH / 32; ++k)
      *reinterpret_cast<uint4*>(tile + canon(t0 + rb * 8 + lr, (4 * k + kc) * 8, DH)) = v[rb][k];
}

// the reverse: canonical tile rows [t0, t0 + 32) → the warp's rows of dst (rows ≥ nvalid skipped)
template <int DH>
__device__ __forceinline__ void warp_canon_to_rows(bf16* dst, long long ld, const bf16* tile, int t0, int nvalid,
                                                   int lane) {
  const int lr = lane & 7, kc = lane >> 3;
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int k = 0; k < DH / 32; ++k) {
      const int r = rb * 8 + lr;
      const uint4 v = *reinterpret_cast<const uint4*>(tile + canon(t0 + r, (4 * k + kc) * 8, DH));
      if (r < nvalid) *reinterpret_cast<uint4*>(dst + r * ld + (4 * k + kc) * 8) = v;
    }
}

__device__ __forceinline__ float dot8_bf16(uint4 a, uint4 b) {
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&b);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(x[i]), q = __bfloat1622float2(y[i]);
    acc = fmaf(p.x, q.x, fmaf(p.y, q.y, acc));
  }
  return acc;
}

template <int DH>
__global__ void __launch_bounds__(kThreads, 2) serve_attn_kernel(ServeAttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int kC = 128;
  constexpr int kKP = 128 * (DH > kC ? DH : kC);     // K tile, then the chunk's P tile
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sV = sQ + 128 * DH;
  bf16* sKP = sV + kC * DH;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKP + kKP);
  uint64_t* bar_a = bars;
  uint64_t* bar_d = bars + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tiles = (a.C + 127) / 128;
  const int hd = blockIdx.x % a.heads;
  const int tile = (blockIdx.x / a.heads) % tiles;
  const int u = blockIdx.x / (a.heads * tiles);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_a, 32 * kWorkers);
    sm100::mbar_init(bar_d, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc<256>(tmem_slot);
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
      const uint32_t aQ = sm100::smem_u32(sQ), aV = sm100::smem_u32(sV), aKP = sm100::smem_u32(sKP);
      uint32_t pa = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      for (int c = 0; c < nchunk; ++c) {
        wait_a();
        mma(T_S, Opnd{aQ, DH, 0}, Opnd{aKP, DH, 0}, DH / 16, kC, false);
        sm100::mma_commit(bar_d);
        wait_a();
        mma(T_O, Opnd{aKP, kC, 0}, Opnd{aV, DH, 1}, kC / 16, DH, c > 0);
        sm100::mma_commit(bar_d);
      }
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float scale = rsqrtf((float)(a.D / a.heads));
    const int npg = a.npg[u];
    const int c_base = tile * 128 + q * 32;                         // the warp's first candidate
    const int nrow = min(32, a.C - c_base);                         // its valid rows
    const bool qrow = lane < nrow;
    const long long r_base = (long long)u * a.C + c_base;
    uint32_t pd = 0;
    auto signal = [&]() { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar_a); };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    // own query rows → sQ, and q·k_own for each of them (lanes lr + 8·kc share a row)
    float s_own;
    {
      const int lr = lane & 7, kc = lane >> 3;
      float part[4];
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        const int r = rb * 8 + lr;
        part[rb] = 0.f;
#pragma unroll
        for (int k = 0; k < DH / 32; ++k) {
          const int col = hd * DH + (4 * k + kc) * 8;
          uint4 qv = make_uint4(0, 0, 0, 0), kv = qv;
          if (r < nrow) {
            qv = *reinterpret_cast<const uint4*>(a.Q + (r_base + r) * a.ldq + col);
            kv = *reinterpret_cast<const uint4*>(a.Kown + (r_base + r) * a.ldown + col);
          }
          *reinterpret_cast<uint4*>(sQ + canon(q * 32 + r, (4 * k + kc) * 8, DH)) = qv;
          part[rb] += dot8_bf16(qv, kv);
        }
        part[rb] += __shfl_xor_sync(0xffffffffu, part[rb], 8);
        part[rb] += __shfl_xor_sync(0xffffffffu, part[rb], 16);
      }
      s_own = 0.f;
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        const float v = __shfl_sync(0xffffffffu, part[rb], lane & 7);
        if ((lane >> 3) == rb) s_own = v;
      }
      s_own = qrow ? s_own * scale : -INFINITY;
    }
    float m = s_own, l = qrow ? 1.f : 0.f;                          // the own key is always visible
    auto visible = [&](int key) { return key < a.nk && (key >= a.ns || a.goff + key >= npg); };
    const bf16* Kb = a.K + u * a.sk + hd * DH;
    const bf16* Vb = a.V + u * a.sv + hd * DH;
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * kC, k0 = c0 + q * 32;
      // the P·V MMA of chunk c-1 has completed (wait_d below): both tiles are free
      warp_rows_to_canon<DH>(sKP, q * 32, Kb + (long long)k0 * a.ldk, a.ldk, a.nk - k0, lane);
      warp_rows_to_canon<DH>(sV, q * 32, Vb + (long long)k0 * a.ldv, a.ldv, a.nk - k0, lane);
      signal();
      wait_d();                                                     // S = Q·Kᵀ
      float cm = -INFINITY;
#pragma unroll 1
      for (int j0 = 0; j0 < kC; j0 += 32) {
        float s[32];
        tmem_row<32>(T_S + lo + j0, s);
#pragma unroll
        for (int v = 0; v < 32; ++v)
          if (visible(c0 + j0 + v)) cm = fmaxf(cm, s[v] * scale);
      }
      const bool grow = qrow && cm > m + kRescale;
      if (__any_sync(0xffffffffu, grow)) {
        const float f = grow ? __expf(m - cm) : 1.f;
        if (grow) { l *= f; m = cm; }
        if (c > 0) {
#pragma unroll 1
          for (int j0 = 0; j0 < DH; j0 += 32) {
            float o[32];
            tmem_row<32>(T_O + lo + j0, o);
#pragma unroll
            for (int v = 0; v < 32; ++v) o[v] *= f;
            tmem_row_st<32>(T_O + lo + j0, o);
          }
        }
      }
#pragma unroll 1
      for (int j0 = 0; j0 < kC; j0 += 32) {
        float s[32];
        tmem_row<32>(T_S + lo + j0, s);
        float add = 0.f;
#pragma unroll
        for (int v = 0; v < 32; ++v) {
          s[v] = (qrow && visible(c0 + j0 + v)) ? __expf(s[v] * scale - m) : 0.f;
          add += s[v];
        }
        l += add;
        store_row(sKP, row, kC, s, 32, j0);                         // P over the (consumed) K tile
      }
      signal();
      wait_d();                                                     // O += P·V
    }
    // epilogue: ctx = (O + p_own·v_own) / l, staged through the (free) tiles for coalesced I/O
    const float rl = l > 0.f ? 1.f / l : 0.f;
    const float p_own = qrow ? __expf(s_own - m) : 0.f;
    warp_rows_to_canon<DH>(sV, q * 32, a.Vown + r_base * a.ldown + hd * DH, a.ldown, nrow, lane);
    __syncwarp();
#pragma unroll 1
    for (int j0 = 0; j0 < DH; j0 += 32) {
      float o[32];
      tmem_row<32>(T_O + lo + j0, o);
#pragma unroll
      for (int cc = 0; cc < 32; cc += 8) {
        const uint4 vv = *reinterpret_cast<const uint4*>(sV + canon(row, j0 + cc, DH));
        const __nv_bfloat162* vp = reinterpret_cast<const __nv_bfloat162*>(&vv);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 w = __bfloat1622float2(vp[i]);
          o[cc + 2 * i] = (o[cc + 2 * i] + p_own * w.x) * rl;
          o[cc + 2 * i + 1] = (o[cc + 2 * i + 1] + p_own * w.y) * rl;
        }
      }
      store_row(sKP, row, DH, o, 32, j0);
    }
    __syncwarp();
    warp_canon_to_rows<DH>(a.ctx + r_base * a.ldc + hd * DH, a.ldc, sKP, q * 32, nrow, lane);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

template <int DH>
int launch_serve(const ServeAttnArgs& a, cudaStream_t st) {
  const int smem = (128 * DH + 128 * DH + 128 * (DH > 128 ? DH : 128)) * 2 + 64;
  smem_attr(serve_attn_kernel<DH>, smem);
  const int tiles = (a.C + 127) / 128;
  launch(serve_attn_kernel<DH>, a.U * tiles * a.heads, kThreads, smem, st, a);
  return (int)cudaGetLastError();
}

// SIMT variant for head widths the tensor-core tile does not take (D/heads ∉ {32, 64, 128}):
// one warp per (candidate row, head); lanes stride the keys for the statistics and split the
// head dims for P·V.
__global__ void serve_attn_simt_kernel(ServeAttnArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float s_q[];                       // [warps][dh]
  const int dh = a.D / a.heads;
  const int wib = threadIdx.x / 32, lane = threadIdx.x & 31;
  const long long task = (long long)blockIdx.x * (blockDim.x / 32) + wib;
  const long long R = (long long)a.U * a.C;
  if (task >= R * a.heads) return;
  const long long r = task / a.heads;
  const int hd = (int)(task % a.heads);
  const int u = (int)(r / a.C);
  float* q = s_q + wib * dh;
  for (int c = lane; c < dh; c += 32) q[c] = __bfloat162float(a.Q[r * a.ldq + hd * dh + c]);
  __syncwarp();
  const float scale = rsqrtf((float)dh);
  const int npg = a.npg[u];
  const bf16* Kb = a.K + u * a.sk + hd * dh;
  const bf16* Vb = a.V + u * a.sv + hd * dh;
  const bf16* ko = a.Kown + r * a.ldown + hd * dh;
  const bf16* vo = a.Vown + r * a.ldown + hd * dh;
  auto score = [&](int j) {               // j == nk: the row's own key
    const bf16* kr = j < a.nk ? Kb + (long long)j * a.ldk : ko;
    float acc = 0.f;
    for (int c = 0; c < dh; ++c) acc = fmaf(q[c], __bfloat162float(kr[c]), acc);
    return acc * scale;
  };
  auto visible = [&](int j) { return j == a.nk || j >= a.ns || a.goff + j >= npg; };
  float m = -INFINITY, l = 0.f;
  for (int j = lane; j <= a.nk; j += 32) {
    if (!visible(j)) continue;
    const float s = score(j);
    const float mn = fmaxf(m, s);
    l = l * __expf(m - mn) + __expf(s - mn);
    m = mn;
  }
  const float M = warp_max(m);
  l = warp_sum(m == -INFINITY ? 0.f : l * __expf(m - M));
  const float rl = 1.f / l;                            // the own key is always visible: l ≥ 1
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int j0 = 0; j0 <= a.nk; j0 += 32) {
    const int j = j0 + lane;
    const float p = (j <= a.nk && visible(j)) ? __expf(score(j) - M) * rl : 0.f;
    const int n = min(32, a.nk + 1 - j0);
    for (int t = 0; t < n; ++t) {
      const float pt = __shfl_sync(0xffffffffu, p, t);
      if (pt == 0.f) continue;
      const int jt = j0 + t;
      const bf16* vr = jt < a.nk ? Vb + (long long)jt * a.ldv : vo;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = lane + 32 * i;
        if (c < dh) o[i] = fmaf(pt, __bfloat162float(vr[c]), o[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = lane + 32 * i;
    if (c < dh) a.ctx[r * a.ldc + hd * dh + c] = __float2bfloat16(o[i]);
  }
}

int serve_attn(const ServeAttnArgs& a, cudaStream_t st) {
  const int dh = a.D / a.heads;
  if (dh == 128) return launch_serve<128>(a, st);
  if (dh == 64) return launch_serve<64>(a, st);
  if (dh == 32) return launch_serve<32>(a, st);
  if (dh > 256) return (int)cudaErrorInvalidValue;
  const long long tasks = (long long)a.U * a.C * a.heads;
  launch(serve_attn_simt_kernel, (unsigned)((tasks + 3) / 4), 128, 4 * dh * sizeof(float), st, a);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ head over candidate rows
// Head of every target row: forward_tensor's head (pkg/src/longrec/model.py:346-362) with the
// cached CLS row and user-side features of the candidate's user (score_with_cache,
// serving.py:160-166), in fp32 like the training head.  A warp takes kHeadRows rows at a time,
// lane j = hidden unit j (+32, …).  W1 / b1 / w2 stay in shared memory for the whole persistent
// kernel (lane j reads column j of W1: conflict-free).  A row group is kHeadRows candidates of ONE
// user.  The head input [t, c, t·c, t·t, u_d] is never materialised: the warp stages its rows' t
// and the user's c and u_d (coalesced), and for every 4 input columns i the 16 W1 words of the
// four segments (rows i, D+i, 2D+i, 3D+i) are loaded once and applied to all kHeadRows rows from
// float4 broadcasts of t (the user's c is folded into the t weights once per group: t·(W_t + c⊙W_tc)
// + t²·W_tt, with t·(w_a + t·w_tt) one FMA pair per input).
constexpr int kHeadRows = 8, kHeadThreads = 512;

template <bool kSmemW>
__global__ void __launch_bounds__(kHeadThreads) serve_head_kernel(ServeHeadArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int D = a.D, d2 = 2 * a.d, HIN = 4 * D + d2, hh = a.hh;
  const int XS = kHeadRows * D + D + d2;                   // per warp: t [kHeadRows][D], c [D], u_d [2d]
  float* sX = sm;
  float* sW = sX + (kHeadThreads / 32) * XS;               // [HIN][hh]
  float* sB = sW + (kSmemW ? HIN * hh : 0);                 // b1 [hh], w2 [hh]
  if (kSmemW)
    for (int i = threadIdx.x; i < HIN * hh; i += blockDim.x) sW[i] = a.w1[i];
  for (int i = threadIdx.x; i < hh; i += blockDim.x) { sB[i] = a.b1[i]; sB[hh + i] = a.w2[i]; }
  const float* W = kSmemW ? sW : a.w1;
  __syncthreads();
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  float* x = sX + wid * XS;
  float* xc = x + kHeadRows * D;
  float* xu = xc + D;
  const float b2 = a.b2[0];
  const int gpu_ = (a.C + kHeadRows - 1) / kHeadRows;      // groups per user
  const long long ngroups = (a.R / a.C) * gpu_;
  for (long long g = (long long)blockIdx.x * nw + wid; g < ngroups; g += (long long)gridDim.x * nw) {
    const int u = (int)(g / gpu_);
    const int c0 = (int)(g % gpu_) * kHeadRows;
    const long long r0 = (long long)u * a.C + c0;
    const int nr = min(kHeadRows, a.C - c0);
    __syncwarp();
    const float4* t = reinterpret_cast<const float4*>(a.x + r0 * D);
    for (int i = lane; i < kHeadRows * D / 4; i += 32)
      reinterpret_cast<float4*>(x)[i] = i < nr * D / 4 ? t[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* c = reinterpret_cast<const float4*>(a.cls + (long long)u * D);
    for (int i = lane; i < D / 4; i += 32) reinterpret_cast<float4*>(xc)[i] = c[i];
    for (int i = lane; i < d2; i += 32) xu[i] = a.ud[(long long)u * d2 + i];
    __syncwarp();
    float zp[kHeadRows];
#pragma unroll
    for (int q = 0; q < kHeadRows; ++q) zp[q] = 0.f;
    for (int j = lane; j < hh; j += 32) {
      // z1 = t·(W_t + diag(c)·W_tc) + (t⊙t)·W_tt + [c·W_c + u_d·W_ud + b1]: the user's c folds into
      // the t weights once per row group, and the bracket is one value per group
      float acc[kHeadRows];
      float kc = sB[j];
#pragma unroll
      for (int q = 0; q < kHeadRows; ++q) acc[q] = 0.f;
#pragma unroll 1
      for (int i = 0; i < D; i += 4) {
        const float4 c4 = *reinterpret_cast<const float4*>(xc + i);
        const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
        float wa[4], wtt[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          wa[e] = fmaf(cv[e], W[(2 * D + i + e) * hh + j], W[(i + e) * hh + j]);
          kc = fmaf(cv[e], W[(D + i + e) * hh + j], kc);
          wtt[e] = W[(3 * D + i + e) * hh + j];
        }
#pragma unroll
        for (int q = 0; q < kHeadRows; ++q) {
          const float4 t4 = *reinterpret_cast<const float4*>(x + q * D + i);
          const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
          float v = acc[q];
#pragma unroll
          for (int e = 0; e < 4; ++e) v = fmaf(tv[e], fmaf(tv[e], wtt[e], wa[e]), v);
          acc[q] = v;
        }
      }
#pragma unroll 1
      for (int i = 0; i < d2; ++i) kc = fmaf(xu[i], W[(4 * D + i) * hh + j], kc);
#pragma unroll
      for (int q = 0; q < kHeadRows; ++q) acc[q] += kc;
      const float w2j = sB[hh + j];
#pragma unroll
      for (int q = 0; q < kHeadRows; ++q) zp[q] = fmaf(gelu_f(acc[q]), w2j, zp[q]);
    }
#pragma unroll
    for (int q = 0; q < kHeadRows; ++q) {
      const float z = warp_sum(zp[q]) + b2;
      if (lane == q && q < nr) {
        const float e = __expf(-fabsf(z));
        a.probs[r0 + q] = z >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
      }
    }
  }
}

void serve_head(const ServeHeadArgs& a, cudaStream_t st) {
  if (!a.R) return;
  if (a.D % 4) { fprintf(stderr, "serve_head: D = %d not a multiple of 4\n", a.D); abort(); }
  const int XS = kHeadRows * a.D + a.D + 2 * a.d;
  const int sx = 4 * ((kHeadThreads / 32) * XS + 2 * a.hh);
  const int sw = 4 * (4 * a.D + 2 * a.d) * a.hh;
  const long long groups = (a.R / a.C) * ((a.C + kHeadRows - 1) / kHeadRows);
  const long long blocks = (groups + kHeadThreads / 32 - 1) / (kHeadThreads / 32);
  const unsigned grid = (unsigned)std::min<long long>(blocks, 148);
  if (sx + sw <= 220 * 1024) {
    smem_attr(serve_head_kernel<true>, sx + sw);
    launch(serve_head_kernel<true>, grid, kHeadThreads, sx + sw, st, a);
  } else {
    smem_attr(serve_head_kernel<false>, sx);
    launch(serve_head_kernel<false>, grid, kHeadThreads, sx, st, a);
  }
}

}  // namespace longer
