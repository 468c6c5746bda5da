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
  int item = a.cand[r];
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

// ------------------------------------------------------------------ cached attention
// One CTA per (user, 128-candidate tile, head).  All queries are target rows (global rank m-1):
// they see every non-pad sequence key and every cached global, plus their own key appended last.
// Exact two-pass softmax; S = Q·K_cacheᵀ on the tensor core (TMEM), the own key in registers.
template <int DH>
__global__ void __launch_bounds__(kThreads, 1) serve_attn_kernel(ServeAttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int kC = 128;
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sK = sQ + 128 * DH;
  bf16* sV = sK + kC * DH;
  bf16* sP = sV + kC * DH;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 128 * kC);
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
      const uint32_t aQ = sm100::smem_u32(sQ), aK = sm100::smem_u32(sK), aV = sm100::smem_u32(sV);
      const uint32_t aP = sm100::smem_u32(sP);
      uint32_t pa = 0;
      auto wait_a = [&]() { sm100::mbar_wait(bar_a, pa); pa ^= 1; sm100::tc_fence_after(); };
      for (int c = 0; c < nchunk; ++c) {
        wait_a();
        mma(T_S, Opnd{aQ, DH, 0}, Opnd{aK, DH, 0}, DH / 16, kC, false);
        sm100::mma_commit(bar_d);
      }
      for (int c = 0; c < nchunk; ++c) {
        wait_a();
        mma(T_S, Opnd{aQ, DH, 0}, Opnd{aK, DH, 0}, DH / 16, kC, false);
        sm100::mma_commit(bar_d);
        wait_a();
        mma(T_O, Opnd{aP, kC, 0}, Opnd{aV, DH, 1}, kC / 16, DH, c > 0);
        sm100::mma_commit(bar_d);
      }
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    const float scale = rsqrtf((float)(a.D / a.heads));
    const int npg = a.npg[u];
    const int cand = tile * 128 + row;
    const bool qrow = cand < a.C;
    const long long qr = (long long)u * a.C + cand;                 // candidate row index
    const bf16* Kb = a.K + u * a.sk + hd * DH;
    const bf16* Vb = a.V + u * a.sv + hd * DH;
    uint32_t pd = 0;
    auto signal = [&]() { sm100::fence_async_smem(); sm100::tc_fence_before(); sm100::mbar_arrive(bar_a); };
    auto wait_d = [&]() { sm100::mbar_wait(bar_d, pd); pd ^= 1; sm100::tc_fence_after(); };
    // own query / key / value rows
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (qrow) v = *reinterpret_cast<const uint4*>(a.Q + qr * a.ldq + hd * DH + c);
      *reinterpret_cast<uint4*>(sQ + canon(row, c, DH)) = v;
    }
    float s_own = -INFINITY;
    if (qrow) {
      float acc = 0.f;
      const bf16* qp = a.Q + qr * a.ldq + hd * DH;
      const bf16* kp = a.Kown + qr * a.ldown + hd * DH;
      for (int c = 0; c < DH; ++c) acc = fmaf(__bfloat162float(qp[c]), __bfloat162float(kp[c]), acc);
      s_own = acc * scale;
    }
    float m = s_own, l = qrow ? 1.f : 0.f;                          // the own key is always visible
    auto visible = [&](int key) { return key < a.nk && (key >= a.ns || a.goff + key >= npg); };
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * kC;
#pragma unroll
      for (int cc = 0; cc < DH; cc += 8) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (c0 + row < a.nk) v = *reinterpret_cast<const uint4*>(Kb + (long long)(c0 + row) * a.ldk + cc);
        *reinterpret_cast<uint4*>(sK + canon(row, cc, DH)) = v;
      }
      signal();
      wait_d();
#pragma unroll 1
      for (int j0 = 0; j0 < kC; j0 += 32) {
        float s[32];
        tmem_row<32>(T_S + lo + j0, s);
        if (!qrow) continue;
        float cm = -INFINITY;
#pragma unroll
        for (int v = 0; v < 32; ++v) {
          s[v] = visible(c0 + j0 + v) ? s[v] * scale : -INFINITY;
          cm = fmaxf(cm, s[v]);
        }
        if (cm == -INFINITY) continue;
        const float mn = fmaxf(m, cm);
        float add = 0.f;
#pragma unroll
        for (int v = 0; v < 32; ++v) add += __expf(s[v] - mn);
        l = l * __expf(m - mn) + add;
        m = mn;
      }
    }
    const float rl = l > 0.f ? 1.f / l : 0.f;
    for (int c = 0; c < nchunk; ++c) {
      const int c0 = c * kC;
#pragma unroll
      for (int cc = 0; cc < DH; cc += 8) {
        uint4 kv = make_uint4(0, 0, 0, 0), vv = kv;
        if (c0 + row < a.nk) {
          kv = *reinterpret_cast<const uint4*>(Kb + (long long)(c0 + row) * a.ldk + cc);
          vv = *reinterpret_cast<const uint4*>(Vb + (long long)(c0 + row) * a.ldv + cc);
        }
        *reinterpret_cast<uint4*>(sK + canon(row, cc, DH)) = kv;
        *reinterpret_cast<uint4*>(sV + canon(row, cc, DH)) = vv;
      }
      signal();
      wait_d();
#pragma unroll 1
      for (int j0 = 0; j0 < kC; j0 += 32) {
        float s[32];
        tmem_row<32>(T_S + lo + j0, s);
#pragma unroll
        for (int v = 0; v < 32; ++v) s[v] = (qrow && visible(c0 + j0 + v)) ? __expf(s[v] * scale - m) * rl : 0.f;
        store_row(sP, row, kC, s, 32, j0);
      }
      signal();
      wait_d();
    }
    float o[DH];
    tmem_row<DH>(T_O + lo, o);
    if (qrow) {
      const float p_own = __expf(s_own - m) * rl;
      const bf16* vp = a.Vown + qr * a.ldown + hd * DH;
      bf16* dst = a.ctx + qr * a.ldc + hd * DH;
#pragma unroll
      for (int cc = 0; cc < DH; cc += 8) {
        float w[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) w[v] = o[cc + v] + p_own * __bfloat162float(vp[cc + v]);
        uint4 pk;
        pk.x = sm100::pack_bf16(w[0], w[1]); pk.y = sm100::pack_bf16(w[2], w[3]);
        pk.z = sm100::pack_bf16(w[4], w[5]); pk.w = sm100::pack_bf16(w[6], w[7]);
        *reinterpret_cast<uint4*>(dst + cc) = pk;
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc<256>(tmem);
}

template <int DH>
int launch_serve(const ServeAttnArgs& a, cudaStream_t st) {
  const int smem = (128 * DH + 2 * 128 * DH + 128 * 128) * 2 + 64;
  smem_attr(serve_attn_kernel<DH>, 227 * 1024);
  const int tiles = (a.C + 127) / 128;
  launch(serve_attn_kernel<DH>, a.U * tiles * a.heads, kThreads, std::max(smem, 116 * 1024), st, a);
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
// head of forward_tensor (pkg/src/longrec/model.py:346-362) with the cached CLS row and user-side
// features of the candidate's user (score_with_cache, serving.py:160-166).
__global__ void serve_head_kernel(ServeHeadArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float s_in[];
  const long long r = blockIdx.x;
  const int u = (int)(r / a.C);
  const int D = a.D, HIN = 4 * D + 2 * a.d;
  const float* t = a.x + r * D;
  const float* c = a.cls + (long long)u * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float tv = t[i], cv = c[i];
    s_in[i] = tv; s_in[D + i] = cv; s_in[2 * D + i] = tv * cv; s_in[3 * D + i] = tv * tv;
  }
  for (int i = threadIdx.x; i < 2 * a.d; i += blockDim.x) s_in[4 * D + i] = a.ud[(long long)u * 2 * a.d + i];
  __syncthreads();
  float* s_h = s_in + HIN;
  const int wid = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  for (int j = wid; j < a.hh; j += nw) {
    float acc = 0.f;
    for (int i = lane; i < HIN; i += 32) acc = fmaf(s_in[i], __ldg(a.w1 + i * a.hh + j), acc);
    acc = warp_sum(acc) + a.b1[j];
    if (lane == 0) s_h[j] = gelu_f(acc);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float acc = 0.f;
    for (int j = threadIdx.x; j < a.hh; j += 32) acc = fmaf(s_h[j], a.w2[j], acc);
    acc = warp_sum(acc);
    if (threadIdx.x == 0) {
      const float z = acc + a.b2[0];
      const float e = __expf(-fabsf(z));
      a.probs[r] = z >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
    }
  }
}

void serve_head(const ServeHeadArgs& a, cudaStream_t st) {
  const int smem = 4 * (4 * a.D + 2 * a.d + a.hh);
  if (a.R) launch(serve_head_kernel, (unsigned)a.R, 128, smem, st, a);
}

}  // namespace longer
