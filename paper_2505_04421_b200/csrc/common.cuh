// common.cuh — shared device helpers: GELU, warp reductions, bf16 access, visibility rule.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

namespace longer {

typedef __nv_bfloat16 bf16;

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the library is launched with programmatic stream serialisation: the next kernel
// of the step may be scheduled while this one drains, runs its prologue (barrier init, TMEM
// allocation, tensor-map prefetch), then blocks in pdl_wait() until its predecessor has finished
// and its writes are visible.  Rules that keep this safe: pdl_wait() precedes every global-memory
// access of a kernel; kernels that allocate TMEM call pdl_trigger() only after their allocation (a
// waiting dependent never holds TMEM that a not-yet-allocated predecessor CTA needs).
// LONGER_PDL=0 disables the attribute (plain stream order).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Tuning / ablation switches (environment, LONGER_*).  Read into thread-local storage at every
// C-ABI entry (refresh_knobs), so a test can toggle them between calls and two threads driving
// the library never share them.  Defaults are the measured-best settings.
struct Knobs {
  int pdl = 1;             // LONGER_PDL: programmatic dependent launch
  int pdl_fence = 15;      // LONGER_PDL_FENCE: full (non-programmatic) dependencies around the big kernels:
                           // bit 0 into the fused front-end kernels, bit 1 out of them, bits 2 / 3 the
                           // same for the cross-attention kernels, bits 4 / 5 for the GEMMs.  An early
                           // (programmatic) launch parks the dependent grid's CTAs on SMs that the
                           // predecessor's tail and the side stream's kernels could use: measured at
                           // c2-inner, 47 (all but into the GEMMs) 1.264-1.280 ms, 15: 1.291, 0: 1.37,
                           // PDL off: 1.30; bits 6 / 7 (every other kernel) cost +8 / +20 us; without
                           // bit 0 +18 us, without bit 3 +55 us, bits 1 and 2 within noise.  With the
                           // GEMMs triggering their dependents only after their last MMA issue
                           // (gemm_late_trigger), 15 (no fence out of the GEMMs) gives 1.245 ms
                           // (47: 1.279); c5 6.65 -> 6.60, c2-concat 0.967 -> 0.941, c1 0.324 -> 0.304
  int prio = 1;            // LONGER_PRIO: side stream at the lowest launch priority
  int side = 1;            // LONGER_SIDE: weight-gradient side stream
  int fused = 1;           // LONGER_FUSED: fused front-end kernels
  int attn_tc = 1;         // LONGER_ATTN_TC: tensor-core attention
  int attn_tma = 1;        // LONGER_ATTN_TMA: K/V by TMA
  int attn_pack = 1;       // LONGER_ATTN_PACK: 0 off, 1 backward, 2 forward too
  int attn_short = 1;      // LONGER_ATTN_SHORT: double-buffered cross-attention backward (nq <= 64)
  int absorb_kv = 1;       // LONGER_ABSORB_KV: cross-layer K/V projections absorbed into the query rows
  int attn_kvs = 1;        // LONGER_ATTN_KVS: one shared K = V tile per key chunk when keys are values
  int attn_bwd_t = 1;      // LONGER_ATTN_BWD_T: keys-as-rows cross-attention backward (keys = values)
  int glob_side = 1;       // LONGER_GLOB_SIDE: global-token backward chain on the side stream
  int head_rows = 1;       // LONGER_HEAD_ROWS: last block's row-wise tail on the two head rows
  int gemm_stage = 1;      // LONGER_GEMM_STAGE: smem-staged GEMM epilogue stores
  int split_items = 37;    // LONGER_SPLIT_ITEMS: split-K work-item target of the weight gradients
                           // (37 vs 74 at the end of round 2: c2 equal over 4 A/B pairs, c5 -15 us)
  int gemm_min_tiles = 0;    // LONGER_GEMM_MIN_TILES: fewest items a wider GEMM tile must give
                             // (0: 60 for K, N >= 256 — wide tiles re-read A less — else 200)
  int fe_grid = 0;         // LONGER_FE_GRID: cap on the fused front-end grids (0: the full machine)
  int item_smem = 1;       // LONGER_ITEM_SMEM: item-table gradient staged in shared memory
  int fe_kn_global = 1;    // LONGER_FE_KN_GLOBAL: fe_fwd's cross-LN1 params from L1 when that buys a fourth slot
  int gemm_late_trigger = 1;  // LONGER_GEMM_LATE_TRIGGER: GEMM dependents launch after its last MMA issue
  int ln256 = 1;           // LONGER_LN256: pipelined warp-per-row LN backward for 256-wide K/V rows
  int fe_split = 1;        // LONGER_FE_SPLIT: fe_mlp_bwd tile ranges across column blocks (0 off, 1 when
                           // it shortens the longest CTA by > 25%, 2 always)
};

inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

inline Knobs read_knobs() {
  Knobs k;
  k.pdl = env_int("LONGER_PDL", 1);
  k.pdl_fence = env_int("LONGER_PDL_FENCE", 15);
  k.prio = env_int("LONGER_PRIO", 1);
  k.side = env_int("LONGER_SIDE", 1);
  k.fused = env_int("LONGER_FUSED", 1);
  k.attn_tc = env_int("LONGER_ATTN_TC", 1);
  k.attn_tma = env_int("LONGER_ATTN_TMA", 1);
  k.attn_pack = env_int("LONGER_ATTN_PACK", 1);
  k.attn_short = env_int("LONGER_ATTN_SHORT", 1);
  k.absorb_kv = env_int("LONGER_ABSORB_KV", 1);
  k.attn_kvs = env_int("LONGER_ATTN_KVS", 1);
  k.attn_bwd_t = env_int("LONGER_ATTN_BWD_T", 1);
  k.glob_side = env_int("LONGER_GLOB_SIDE", 1);
  k.head_rows = env_int("LONGER_HEAD_ROWS", 1);
  k.gemm_stage = env_int("LONGER_GEMM_STAGE", 1);
  k.split_items = env_int("LONGER_SPLIT_ITEMS", 37);
  k.gemm_min_tiles = env_int("LONGER_GEMM_MIN_TILES", 0);
  k.fe_grid = env_int("LONGER_FE_GRID", 0);
  k.item_smem = env_int("LONGER_ITEM_SMEM", 1);
  k.fe_split = env_int("LONGER_FE_SPLIT", 1);
  k.ln256 = env_int("LONGER_LN256", 1);
  k.gemm_late_trigger = env_int("LONGER_GEMM_LATE_TRIGGER", 1);
  k.fe_kn_global = env_int("LONGER_FE_KN_GLOBAL", 1);
  if (k.split_items < 1) k.split_items = 1;
  if (k.gemm_min_tiles < 0) k.gemm_min_tiles = 0;
  return k;
}

inline thread_local Knobs g_knobs = read_knobs();
inline void refresh_knobs() { g_knobs = read_knobs(); }

// Raise a kernel's dynamic shared-memory limit to the opt-in maximum (227 KB less its static
// shared memory), once per (kernel, device): the limit is a per-device setting, so a process
// driving several GPUs raises it on each.  (`bytes` only documents the launch's need: the limit is
// not an occupancy hint, and one limit serves every launch shape of the kernel.)
inline void smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  (void)bytes;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({kernel, dev}).second) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024 - static_cast<int>(fa.sharedSizeBytes));
  }
}
template <typename... KArgs>
inline void smem_attr(void (*kernel)(KArgs...), int bytes) {
  smem_attr(reinterpret_cast<const void*>(kernel), bytes);
}

// The weight-gradient side streams (longer.cu, one per device and driving thread) launch at the
// lowest priority and everything else at the highest, so the block scheduler serves the critical
// dX chain first when both are ready.
inline thread_local cudaStream_t g_side_streams[16] = {};
inline bool is_side_stream(cudaStream_t st) {
  if (!st) return false;
  for (cudaStream_t s : g_side_streams)
    if (s == st) return true;
  return false;
}

inline void launch_priorities(int& lo, int& hi) {
  static int l = 0, h = 0;
  static std::once_flag once;
  std::call_once(once, [] { cudaDeviceGetStreamPriorityRange(&l, &h); });
  lo = l;
  hi = g_knobs.prio ? h : l;                   // LONGER_PRIO=0: all launches at the default priority
}

// PDL fences: a launch flagged `fence_in` gets a full dependency on its predecessor; one flagged
// `fence_out` makes the next launch on its stream do so (see Knobs::pdl_fence)
inline thread_local cudaStream_t g_fence_stream = nullptr;
inline thread_local bool g_fence_pending = false;
enum : int { kFenceNone = 0, kFenceFrontIn = 1, kFenceFrontOut = 2, kFenceAttnIn = 4, kFenceAttnOut = 8,
             kFenceGemmIn = 16, kFenceGemmOut = 32, kFenceOtherIn = 64, kFenceOtherOut = 128 };

inline thread_local int g_launch_fence = 0;   // set by a launcher for its next launch() call
template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  const int fence = (g_launch_fence ? g_launch_fence : (kFenceOtherIn | kFenceOtherOut)) & g_knobs.pdl_fence;
  g_launch_fence = 0;
  bool pdl = g_knobs.pdl != 0;
  if (g_fence_pending && g_fence_stream == st) { pdl = false; g_fence_pending = false; }
  if (fence & (kFenceFrontIn | kFenceAttnIn | kFenceGemmIn | kFenceOtherIn)) pdl = false;
  if (fence & (kFenceFrontOut | kFenceAttnOut | kFenceGemmOut | kFenceOtherOut)) { g_fence_pending = true; g_fence_stream = st; }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  int lo = 0, hi = 0;
  launch_priorities(lo, hi);
  cudaLaunchAttribute at[2];
  int n = 0;
  if (hi != lo) {
    at[n].id = cudaLaunchAttributePriority;
    at[n].val.priority = is_side_stream(st) ? lo : hi;
    ++n;
  }
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr float kGeluC = 0.7978845608028654f;  // sqrt(2/pi)   (pkg/src/longrec/tensors.py:36)
constexpr float kGeluA = 0.044715f;            //              (pkg/src/longrec/tensors.py:37)
constexpr float kLnEps = 1e-12f;               //              (pkg/src/longrec/tensors.py:39)
constexpr float kProbEps = 1e-12f;             //              (pkg/src/longrec/tensors.py:38)

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh-GELU (pkg/src/longrec/tensors.py:292-304), written as FFMA chains:
//   u = x·c(1 + a x²),  t = tanh(u),  gelu = h + h·t (h = x/2),
//   gelu' = (1 + t)/2 + h (1 − t²) c (1 + 3a x²)
__device__ __forceinline__ float gelu_f(float x) {
  const float x2 = x * x;
  const float t = tanh_fast(x * fmaf(x2, kGeluC * kGeluA, kGeluC));
  const float h = 0.5f * x;
  return fmaf(h, t, h);
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float x2 = x * x;
  const float t = tanh_fast(x * fmaf(x2, kGeluC * kGeluA, kGeluC));
  const float h = 0.5f * x;
  return fmaf(h * fmaf(-t, t, 1.f), fmaf(x2, 3.f * kGeluC * kGeluA, kGeluC), fmaf(0.5f, t, 0.5f));
}
// both at once: returns gelu(x), writes gelu'(x)
__device__ __forceinline__ float gelu_and_grad(float x, float& grad) {
  const float x2 = x * x;
  const float t = tanh_fast(x * fmaf(x2, kGeluC * kGeluA, kGeluC));
  const float h = 0.5f * x;
  grad = fmaf(h * fmaf(-t, t, 1.f), fmaf(x2, 3.f * kGeluC * kGeluA, kGeluC), fmaf(0.5f, t, 0.5f));
  return fmaf(h, t, h);
}

// tanh-GELU of two values in packed f16x2 arithmetic (half the instructions of the fp32 form;
// f16 keeps 11 significant bits, more than the bf16 operands the result feeds):
// returns f16x2 {gelu(lo), gelu(hi)}
__device__ __forceinline__ uint32_t gelu2_f16(float lo, float hi) {
  uint32_t x, x2, t, u, th, hh, g;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(x) : "f"(hi), "f"(lo));
  // constants: c = sqrt(2/pi) = 0x3A62, c*a = 0.0356774 = 0x2891, 0.5 = 0x3800 (f16, both halves)
  asm("mul.rn.f16x2 %0, %1, %1;" : "=r"(x2) : "r"(x));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(t) : "r"(x2), "r"(0x28912891u), "r"(0x3A623A62u));
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(u) : "r"(x), "r"(t));
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(th) : "r"(u));
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(hh) : "r"(x), "r"(0x38003800u));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(g) : "r"(hh), "r"(th), "r"(hh));
  return g;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float ldf(const float* p) { return *p; }
__device__ __forceinline__ float ldf(const bf16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void stf(float* p, float v) { *p = v; }
__device__ __forceinline__ void stf(bf16* p, float v) { *p = __float2bfloat16(v); }

// Visibility rule of the hybrid attention (pkg/src/longrec/attention.py:49-87 with the
// metadata of pkg/src/longrec/model.py:275-293), for every query strategy:
//   queries: i < k → sequence query at merged group qgroup(i);  i >= k → global of rank i-k
//   keys:    j < ns → sequence key;  j >= ns → global of rank j-ns
//     cross layer (self_keys = 0): sequence key j is merged group j (ns = G)
//     self layers (self_keys = 1): sequence key j is sequence query j (ns = k)
//   a merged group is pad iff group < npg (pad groups form a prefix of the left-padded grid).
// qg = this sample's sorted query groups (nullptr: "recent", G-k+i); learn = the "learnable" bank
// (every bank row sits at the top grid position and is never pad).
struct VisRule {
  int k, G, ns, goff, npg;
  const int32_t* qg;
  int learn, self_keys;
  __device__ __forceinline__ int qgroup(int i) const { return learn ? G - 1 : (qg ? qg[i] : G - k + i); }
  __device__ __forceinline__ bool qpad(int i) const { return !learn && qgroup(i) < npg; }
  // number of pad sequence queries (always the first ones: the query groups are sorted)
  __device__ __forceinline__ int jpad() const { return learn ? 0 : max(0, k - (G - npg)); }
  __device__ __forceinline__ bool operator()(int i, int j) const {
    if (i < k) {
      if (qpad(i) || j >= ns) return false;
      if (self_keys) return !qpad(j) && qgroup(j) <= qgroup(i);
      return j >= npg && j <= qgroup(i);
    }
    if (j < ns) return self_keys ? !qpad(j) : j >= npg;
    return (j - ns) <= (i - k);
  }
};

}  // namespace longer
