// longer.cu — C ABI (include/longer.h) and the native step orchestrator.
//
// One call runs a whole batch through the LONGER encoder on the caller's stream (plus a side
// stream for work off the critical chain, joined before return):
//   fused front-end (featuriser → token MLP → InnerTrans, frontend.cu) ‖ global tokens → cross
//   block → N self blocks → head + BCE  (forward, pkg/src/longrec/model.py:307-363)
// and, for training, the exact reverse sweep (pkg/src/longrec/tensors.py:141-175) with the weight
// gradients on the side stream.  Row-level contractions go through the tcgen05 GEMM (gemm.cu),
// attention through attn_tc.cu, the rest through ops.cu.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gemm.cuh"
#include "longer.h"
#include "ops.cuh"
#include "frontend.cuh"
#include "serve.cuh"
#include <algorithm>
#include <cstdlib>

namespace longer {
namespace {

thread_local std::string g_err;

// Timing probes (longer_set_probe): optional CUDA events recorded around the fused kernels, on the
// launching stream (graph-capturable), so callers can time one kernel inside a whole step.
enum Phase { PH_FE_FWD = 0, PH_FE_INNER_BWD = 1, PH_FE_MLP_BWD = 2, PH_XATTN_FWD = 3, PH_XATTN_BWD = 4,
             PH_FWD_ROWS = 5, PH_BWD_ROWS = 6, PH_N = 7 };
thread_local cudaEvent_t g_probe[PH_N][2] = {};   // set by longer_set_probe on the driving thread

// Early-gradient event (longer_set_grad_event): recorded once grads[cross, total) are final.
thread_local cudaEvent_t g_grad_event = nullptr;

// (inside a stream capture a plain record is a capture-internal node other streams may wait on)
void record_event(cudaEvent_t ev, cudaStream_t st) { cudaEventRecord(ev, st); }

void probe(int ph, int which, cudaStream_t st) {
  // External record: inside stream capture this becomes a real event-record node (a plain
  // cudaEventRecord would only be a capture-internal dependency marker).
  if (!g_probe[ph][which]) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(g_probe[ph][which], st, cudaEventRecordExternal);
  else cudaEventRecord(g_probe[ph][which], st);
}

// Side stream for the weight-gradient branch: dW GEMMs and bias column sums only feed the
// gradient buffer, so they run beside the critical dX chain (fork after their inputs exist, one
// join at the end of the call).  Inside stream capture the fork/join become graph edges.
// LONGER_SIDE=0 runs everything on the caller's stream.
struct Side {
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, mark_ev = nullptr;
};
thread_local Side g_side[16];     // per device and driving thread: calls never share events

cudaStream_t side_stream(cudaStream_t main) {
  if (!g_knobs.side) return main;
  int dev = 0;
  cudaGetDevice(&dev);
  Side& sd = g_side[dev & 15];
  if (!sd.s) {
    cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking);
    g_side_streams[dev & 15] = sd.s;
    cudaEventCreateWithFlags(&sd.fork_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&sd.join_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&sd.mark_ev, cudaEventDisableTiming);
    sd.dev = dev;
  }
  return sd.s;
}

// side stream waits for everything enqueued on main so far
void fork_side(cudaStream_t main, cudaStream_t side) {
  if (side == main) return;
  int dev = 0;
  cudaGetDevice(&dev);
  Side& sd = g_side[dev & 15];
  cudaEventRecord(sd.fork_ev, main);
  cudaStreamWaitEvent(side, sd.fork_ev, 0);
}

// main waits for everything enqueued on the side stream so far
void join_side(cudaStream_t main, cudaStream_t side) {
  if (side == main) return;
  int dev = 0;
  cudaGetDevice(&dev);
  Side& sd = g_side[dev & 15];
  cudaEventRecord(sd.join_ev, side);
  cudaStreamWaitEvent(main, sd.join_ev, 0);
}

// a point on the side stream that main waits for later (mark_side now, wait_mark at the consumer)
void mark_side(cudaStream_t main, cudaStream_t side) {
  if (side == main) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaEventRecord(g_side[dev & 15].mark_ev, side);
}
void wait_mark(cudaStream_t main, cudaStream_t side) {
  if (side == main) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStreamWaitEvent(main, g_side[dev & 15].mark_ev, 0);
}

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

// query strategies (config.py QUERY_STRATEGIES order)
enum QueryStrategy { QS_RECENT = 0, QS_UNIFORM = 1, QS_LEARNABLE = 2, QS_RECENT_UNIFORM = 3 };

// ------------------------------------------------------------------ parameter offsets
constexpr int kMaxInner = 8;
constexpr int kMaxSelf = 16;

struct BlockOff {
  long long w_q, b_q, w_k, b_k, w_v, b_v, w_o, b_o, w1, b1, w2, b2, ln1_g, ln1_b, ln2_g, ln2_b;
};

struct ParamOff {
  long long item, act, time, uid, prof, pos, cls;
  long long tok_w, tok_b, seq_w1, seq_b1, seq_w2, seq_b2, lift_w, lift_b, glob_w1, glob_b1, glob_w2, glob_b2;
  BlockOff inner[kMaxInner], cross, self_[kMaxSelf];
  long long qbank;             // "learnable" query bank [k, D] (-1 otherwise)
  long long head_w1, head_b1, head_w2, head_b2;
  long long total;
};

// Same order and shapes as LongRecModel.params() (pkg/src/longrec/model.py:252-263).
ParamOff param_offsets(const LongerDims& d) {
  ParamOff o{};
  long long off = 0;
  auto take = [&](long long n) { long long r = off; off += n; return r; };
  const long long D = (long long)d.K * d.d, F = d.d_item + d.d_act + d.d_time;
  o.item = take((long long)d.vocab * d.d_item);
  o.act = take((long long)d.n_actions * d.d_act);
  o.time = take((long long)d.n_time_buckets * d.d_time);
  o.uid = take((long long)d.n_users * d.d);
  o.prof = take((long long)d.n_profiles * d.d);
  o.pos = take((long long)d.L * d.d);
  o.cls = take((long long)(d.m - 2) * D);
  o.tok_w = take(F * d.d); o.tok_b = take(d.d);
  o.seq_w1 = take(d.d * 2 * D); o.seq_b1 = take(2 * D);
  o.seq_w2 = take(2 * D * d.d); o.seq_b2 = take(d.d);
  o.lift_w = take(d.d * D); o.lift_b = take(D);
  o.glob_w1 = take(D * 2 * D); o.glob_b1 = take(2 * D);
  o.glob_w2 = take(2 * D * D); o.glob_b2 = take(D);
  auto block = [&](long long w) {
    BlockOff b;
    b.w_q = take(w * w); b.b_q = take(w); b.w_k = take(w * w); b.b_k = take(w);
    b.w_v = take(w * w); b.b_v = take(w); b.w_o = take(w * w); b.b_o = take(w);
    b.w1 = take(w * 4 * w); b.b1 = take(4 * w); b.w2 = take(4 * w * w); b.b2 = take(w);
    b.ln1_g = take(w); b.ln1_b = take(w); b.ln2_g = take(w); b.ln2_b = take(w);
    return b;
  };
  if (d.merge_inner)
    for (int i = 0; i < d.inner_layers; ++i) o.inner[i] = block(d.d);
  o.cross = block(D);
  for (int i = 0; i < d.N; ++i) o.self_[i] = block(D);
  o.qbank = d.query_strategy == QS_LEARNABLE ? take((long long)d.k * D) : -1;
  const long long hin = 4 * D + 2 * d.d;
  o.head_w1 = take(hin * d.head_hidden); o.head_b1 = take(d.head_hidden);
  o.head_w2 = take(d.head_hidden); o.head_b2 = take(1);
  o.total = off;
  return o;
}

int validate(const LongerDims& d) {
  if (d.L < 1 || d.d < 1 || d.K < 1) return fail(LONGER_ECONFIG, "L, d, K must all be >= 1");
  if (d.m < 3) return fail(LONGER_ECONFIG, "m must be >= 3 (UID, at least one CLS, target)");
  if (d.N < 1 || d.k < 1) return fail(LONGER_ECONFIG, "N and k must be >= 1");
  if (d.query_strategy < 0 || d.query_strategy > 3) return fail(LONGER_ECONFIG, "unknown query strategy");
  const int Lp = (d.L + d.K - 1) / d.K * d.K, G = Lp / d.K, D = d.K * d.d;
  if (d.k > G && d.query_strategy != QS_LEARNABLE) return fail(LONGER_ECONFIG, "k exceeds merged length");
  if (d.heads < 1 || D % d.heads) return fail(LONGER_ECONFIG, "D not divisible by heads");
  if (d.d % 8) return fail(LONGER_ECONFIG, "device path needs d % 8 == 0 (16-byte TMA rows)");
  if (D / d.heads > 256) return fail(LONGER_ECONFIG, "head width D/heads must be <= 256");
  if (d.d > 64 || d.d_item + d.d_act + d.d_time > 64) return fail(LONGER_ECONFIG, "d and feature width must be <= 64");
  if (d.n_time_buckets < 1 || d.n_time_buckets > 32) return fail(LONGER_ECONFIG, "n_time_buckets must be in [1, 32]");
  if (d.merge_inner && (d.inner_layers < 1 || d.inner_layers > kMaxInner)) return fail(LONGER_ECONFIG, "inner_layers out of range");
  if (d.merge_inner && d.K > 16) return fail(LONGER_ECONFIG, "InnerTrans group size K must be <= 16");
  if (d.N > kMaxSelf) return fail(LONGER_ECONFIG, "N too large");
  if (d.k + d.m > 256) return fail(LONGER_ECONFIG, "k + m must be <= 256");
  if (d.batch < 1) return fail(LONGER_EDIM, "batch must be >= 1");
  return LONGER_OK;
}

// ------------------------------------------------------------------ workspace plan
struct Bump {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

struct BlockBufs {            // one attention block over the q query rows
  bf16 *qn, *qkv, *ctx, *x1n, *f1, *gf;
  float *m1, *r1, *lse, *x1, *m2, *r2, *out, *ctx32;
  // backward, per block (the weight-gradient side stream reads them while the main stream moves on)
  float *g_dx, *g_dx1n, *g_dx1, *g_dctx, *g_dqn;    // g_dx = dL/d(block output)
  bf16 *g_dx_bf, *g_df1, *g_dx1_bf, *g_dqkv;
};
struct InnerBufs {            // one InnerTrans layer over T tokens
  bf16 *xn, *ctx, *x1n, *f1, *gf;
  float *m1, *r1, *qkv, *probs, *x1, *m2, *r2, *out;
};
struct Packed {               // bf16 / fp32 operand copies of the weights
  bf16 *seq_w1, *seq_w2, *glob_w1, *glob_w2;
  bf16 *in_wqkv[kMaxInner], *in_wo[kMaxInner], *in_w1[kMaxInner], *in_w2[kMaxInner];
  float* in_bqkv[kMaxInner];
  bf16 *c_wq, *c_wkv, *c_wo, *c_w1, *c_w2;
  float* c_bkv;
  bf16 *s_wqkv[kMaxSelf], *s_wo[kMaxSelf], *s_w1[kMaxSelf], *s_w2[kMaxSelf];
  float* s_bqkv[kMaxSelf];
};

struct Plan {
  LongerDims dims;
  void* ws;
  bool fused_fe;   // fused front-end kernel (frontend.cu) for this call
  bool compact_head = false;   // last self block's row-wise tail on the two head rows only
  // cross layer with absorbed K/V projections (heads = 1): scores Q'·knᵀ with Q' = Q·W_kᵀ, context
  // (P·kn)·W_v + b_v — no [K | V] rows over the B·v key rows (absorb_ok)
  bool absorb = false;
  bf16 *xa_qabs, *xa_craw, *xa_dctx_bf, *xa_dqabs;   // Q', P·kn, dL/dctx (bf16), dL/dQ'
  float *xa_craw32, *xa_dC;                           // P·kn (fp32), dL/d(P·kn)
  float *hc_x, *hc_g, *hc_dctx;   // compact [2B, D] buffers of that tail
  bf16 *hc_ctx, *hc_g_bf;
  bf16* wblob;     // its canonical-layout weight blob
  float* proj;     // the embedding tables projected through tok_proj (FrontArgs::proj)
  int B, L, Lp, d, K, G, D, m, k, q, v, N, heads, inner, IL, hh, F, FP, HIN;
  long long T;
  ParamOff po;
  int* status;
  int32_t* npg;
  int32_t* cand0;  // placeholder candidates of a cache build
  int32_t* qg;     // [B, k] query groups (uniform / recent_uniform)
  int32_t* ids;    // [3, B] range-checked uid / profile / candidate item (check_sample_ids)
  int qs;          // query strategy
  Packed pk;
  // tokens
  bf16 *feat, *x0, *a1, *g1;
  float *real, *keep, *h;
  InnerBufs in[kMaxInner];
  float* merged;
  // globals
  float *raw, *td, *glob;
  bf16 *raw_bf, *ga, *gg;
  // cross
  float *O, *mk, *rk;
  bf16 *kn, *KV;
  BlockBufs cb;
  BlockBufs sb[kMaxSelf];
  // head
  float *hin, *z1, *loss_per, *dz, *dz1;
  // backward scratch (query rows; per-block scratch lives in BlockBufs)
  float* dO;
  float* dkn;
  bf16* dKV;
  float *dmerged, *dglob, *draw;
  bf16 *dglob_bf, *dga;
  // backward scratch (tokens)
  float *t_dx, *t_dx1n, *t_dx1, *t_dctx, *t_dxn, *dx0;
  bf16 *t_dx_bf, *t_df1, *t_dx1_bf, *t_dqkv, *dh_bf, *da1, *dx0_bf;
  size_t bytes;
};

void plan_dims(Plan& p, const LongerDims& d, void* ws) {
  p.dims = d;
  p.ws = ws;
  p.B = d.batch; p.L = d.L; p.K = d.K; p.d = d.d;
  p.Lp = (d.L + d.K - 1) / d.K * d.K;
  p.G = p.Lp / d.K; p.D = d.K * d.d; p.m = d.m; p.k = d.k; p.q = d.k + d.m; p.v = p.G + d.m;
  p.N = d.N; p.heads = d.heads; p.inner = d.merge_inner; p.IL = d.merge_inner ? d.inner_layers : 0;
  p.hh = d.head_hidden; p.F = d.d_item + d.d_act + d.d_time; p.FP = (p.F + 7) / 8 * 8;
  p.HIN = 4 * p.D + 2 * d.d;
  p.T = (long long)p.B * p.Lp;
  p.po = param_offsets(d);
  p.qs = d.query_strategy;
}

void take_packed(Plan& p, Bump& a) {
  const int D = p.D, dd = p.d;
  p.pk.seq_w1 = a.take<bf16>(dd * 2 * D); p.pk.seq_w2 = a.take<bf16>(2 * D * dd);
  p.pk.glob_w1 = a.take<bf16>(D * 2 * D); p.pk.glob_w2 = a.take<bf16>(2 * D * D);
  for (int i = 0; i < p.IL; ++i) {
    p.pk.in_wqkv[i] = a.take<bf16>(dd * 3 * dd); p.pk.in_bqkv[i] = a.take<float>(3 * dd);
    p.pk.in_wo[i] = a.take<bf16>(dd * dd); p.pk.in_w1[i] = a.take<bf16>(dd * 4 * dd); p.pk.in_w2[i] = a.take<bf16>(4 * dd * dd);
  }
  p.pk.c_wq = a.take<bf16>(D * D); p.pk.c_wkv = a.take<bf16>(D * 2 * D); p.pk.c_bkv = a.take<float>(2 * D);
  p.pk.c_wo = a.take<bf16>(D * D); p.pk.c_w1 = a.take<bf16>(D * 4 * D); p.pk.c_w2 = a.take<bf16>(4 * D * D);
  for (int i = 0; i < p.N; ++i) {
    p.pk.s_wqkv[i] = a.take<bf16>(D * 3 * D); p.pk.s_bqkv[i] = a.take<float>(3 * D);
    p.pk.s_wo[i] = a.take<bf16>(D * D); p.pk.s_w1[i] = a.take<bf16>(D * 4 * D); p.pk.s_w2[i] = a.take<bf16>(4 * D * D);
  }
}

Plan make_plan(const LongerDims& d, void* ws) {
  Plan p{};
  plan_dims(p, d, ws);
  Bump a{reinterpret_cast<char*>(ws)};
  const long long T = p.T;
  const int B = p.B, D = p.D, q = p.q, v = p.v, m = p.m, dd = p.d;
  const long long Q = (long long)B * q, V = (long long)B * v, M = (long long)B * m;
  p.status = a.take<int>(64);
  p.npg = a.take<int32_t>(B);
  p.cand0 = a.take<int32_t>(B);
  p.qg = a.take<int32_t>((long long)B * d.k);
  p.ids = a.take<int32_t>(3LL * B);
  p.wblob = a.take<bf16>(frontend_blob_bytes(dd, D, p.IL) / 2 + 64);
  p.proj = a.take<float>((long long)(d.vocab + d.n_actions + d.n_time_buckets) * dd);
  take_packed(p, a);
  // tokens
  p.feat = a.take<bf16>(T * p.FP); p.x0 = a.take<bf16>(T * dd);
  p.real = a.take<float>(T); p.keep = a.take<float>(T);
  p.a1 = a.take<bf16>(T * 2 * D); p.g1 = a.take<bf16>(T * 2 * D);
  p.h = a.take<float>(T * dd);
  for (int i = 0; i < p.IL; ++i) {
    InnerBufs& b = p.in[i];
    b.xn = a.take<bf16>(T * dd); b.m1 = a.take<float>(T); b.r1 = a.take<float>(T);
    b.qkv = a.take<float>(T * 3 * dd); b.probs = a.take<float>(T * d.K); b.ctx = a.take<bf16>(T * dd);
    b.x1 = a.take<float>(T * dd); b.x1n = a.take<bf16>(T * dd); b.m2 = a.take<float>(T); b.r2 = a.take<float>(T);
    b.f1 = a.take<bf16>(T * 4 * dd); b.gf = a.take<bf16>(T * 4 * dd); b.out = a.take<float>(T * dd);
  }
  p.merged = p.IL ? p.in[p.IL - 1].out : p.h;
  // globals
  p.raw = a.take<float>(M * D); p.raw_bf = a.take<bf16>(M * D); p.td = a.take<float>((long long)B * dd);
  p.ga = a.take<bf16>(M * 2 * D); p.gg = a.take<bf16>(M * 2 * D); p.glob = a.take<float>(M * D);
  // cross
  p.O = a.take<float>(Q * D);
  p.kn = a.take<bf16>(V * D); p.mk = a.take<float>(V); p.rk = a.take<float>(V);
  p.KV = a.take<bf16>(V * 2 * D);
  auto block_bufs = [&](BlockBufs& b, int qkv_cols) {
    b.qn = a.take<bf16>(Q * D); b.m1 = a.take<float>(Q); b.r1 = a.take<float>(Q);
    b.qkv = a.take<bf16>(Q * qkv_cols); b.ctx = a.take<bf16>(Q * D); b.lse = a.take<float>(Q * p.heads); b.ctx32 = a.take<float>(Q * D);
    b.x1 = a.take<float>(Q * D); b.x1n = a.take<bf16>(Q * D); b.m2 = a.take<float>(Q); b.r2 = a.take<float>(Q);
    b.f1 = a.take<bf16>(Q * 4 * D); b.gf = a.take<bf16>(Q * 4 * D); b.out = a.take<float>(Q * D);
    b.g_dx = a.take<float>(Q * D); b.g_dx1n = a.take<float>(Q * D); b.g_dx1 = a.take<float>(Q * D);
    b.g_dctx = a.take<float>(Q * D); b.g_dqn = a.take<float>(Q * D);
    b.g_dx_bf = a.take<bf16>(Q * D); b.g_df1 = a.take<bf16>(Q * 4 * D); b.g_dx1_bf = a.take<bf16>(Q * D);
    b.g_dqkv = a.take<bf16>(Q * qkv_cols);
  };
  block_bufs(p.cb, D);
  for (int i = 0; i < p.N; ++i) block_bufs(p.sb[i], 3 * D);
  p.xa_qabs = a.take<bf16>(Q * D); p.xa_craw = a.take<bf16>(Q * D); p.xa_dctx_bf = a.take<bf16>(Q * D);
  p.xa_dqabs = a.take<bf16>(Q * D); p.xa_craw32 = a.take<float>(Q * D); p.xa_dC = a.take<float>(Q * D);
  // head
  p.hin = a.take<float>((long long)B * p.HIN); p.z1 = a.take<float>((long long)B * p.hh);
  p.loss_per = a.take<float>(B); p.dz = a.take<float>(B); p.dz1 = a.take<float>((long long)B * p.hh);
  p.hc_x = a.take<float>(2LL * B * D); p.hc_g = a.take<float>(2LL * B * D); p.hc_dctx = a.take<float>(2LL * B * D);
  p.hc_ctx = a.take<bf16>(2LL * B * D); p.hc_g_bf = a.take<bf16>(2LL * B * D);
  // backward (query rows)
  p.dO = a.take<float>(Q * D);
  p.dkn = a.take<float>(V * D); p.dKV = a.take<bf16>(V * 2 * D);
  p.dmerged = a.take<float>(T * dd); p.dglob = a.take<float>(M * D); p.draw = a.take<float>(M * D);
  p.dglob_bf = a.take<bf16>(M * D); p.dga = a.take<bf16>(M * 2 * D);
  // backward (tokens)
  if (p.IL) {
    p.t_dx = a.take<float>(T * dd); p.t_dx1n = a.take<float>(T * dd); p.t_dx1 = a.take<float>(T * dd);
    p.t_dctx = a.take<float>(T * dd); p.t_dxn = a.take<float>(T * dd);
    p.t_dx_bf = a.take<bf16>(T * dd); p.t_df1 = a.take<bf16>(T * 4 * dd); p.t_dx1_bf = a.take<bf16>(T * dd);
    p.t_dqkv = a.take<bf16>(T * 3 * dd);
  }
  p.dh_bf = a.take<bf16>(T * dd); p.da1 = a.take<bf16>(T * 2 * D);
  p.dx0 = a.take<float>(T * dd); p.dx0_bf = a.take<bf16>(T * dd);
  p.bytes = a.off + 256;
  return p;
}

// ------------------------------------------------------------------ helpers
struct Ctx {
  const Plan& p;
  const float* P;       // fp32 params
  float* G;             // fp32 grads
  cudaStream_t st;
  int rc = 0;
  const float* w(long long off) const { return P + off; }
  float* g(long long off) const { return G + off; }
};

// On failure: the innermost failing call (with the CUDA error text) first, then its callers.
#define TRY(expr)                                                                         \
  do {                                                                                    \
    int _rc = (expr);                                                                     \
    if (_rc) {                                                                            \
      if (g_err.empty()) {                                                                \
        g_err = std::string(#expr) + ": " + cudaGetErrorString((cudaError_t)_rc);         \
      } else {                                                                            \
        g_err += std::string(" | in ") + #expr;                                           \
      }                                                                                   \
      return LONGER_ECUDA;                                                                \
    }                                                                                     \
  } while (0)

// C[M,N] (=|+=) epi(A[M,K]·B[K,N]); majors: a_mn / b_mn as in gemm.cuh
GemmArgs G_(const void* A, int lda, int amn, const void* B, int ldb, int bmn, long long M, int N, long long K) {
  GemmArgs g;
  g.A = A; g.lda = lda; g.a_mn_major = amn; g.B = B; g.ldb = ldb; g.b_mn_major = bmn;
  g.M = (int)M; g.N = N; g.K = (int)K; g.flags = 0;
  return g;
}

// Y = X·W (+bias) variants
int lin_fwd(cudaStream_t st, const bf16* X, int ldx, long long rows, const bf16* W, int in, int out, const float* bias,
            uint32_t flags, float* C, bf16* Cbf, bf16* pre, const float* resid = nullptr, int ldr = 0,
            const float* rowmask = nullptr) {
  GemmArgs g = G_(X, ldx, 0, W, out, 1, rows, out, in);
  g.flags = flags | (bias ? EPI_BIAS : 0u) | (C ? EPI_OUT_F32 : 0u) | (Cbf ? EPI_OUT_BF16 : 0u) |
            (resid ? EPI_RESID : 0u) | (rowmask ? EPI_ROWMASK : 0u);
  g.bias = bias; g.C = C; g.ldc = out; g.C_bf16 = Cbf; g.ldc_bf = out; g.pre_bf16 = pre;
  g.resid = resid; g.ldr = ldr; g.rowmask = rowmask;
  return gemm_launch(g, st);
}

// dX = dY·Wᵀ  (W stored [in, out] row-major = [N][K] K-major B), optional GELU' epilogue
int lin_dx(cudaStream_t st, const bf16* dY, int lddy, long long rows, const bf16* W, int ldw, int in, int out,
           float* C, int ldc, bf16* Cbf, int ldcbf, const bf16* gelu_pre = nullptr, const float* rowmask = nullptr) {
  GemmArgs g = G_(dY, lddy, 0, W, ldw, 0, rows, in, out);
  g.flags = (C ? EPI_OUT_F32 : 0u) | (Cbf ? EPI_OUT_BF16 : 0u) | (gelu_pre ? EPI_GELU_BWD : 0u) |
            (rowmask ? EPI_ROWMASK : 0u);
  g.C = C; g.ldc = ldc; g.C_bf16 = Cbf; g.ldc_bf = ldcbf; g.pre_bf16 = const_cast<bf16*>(gelu_pre);
  g.rowmask = rowmask;
  return gemm_launch(g, st);
}

// dW[in, out] += Xᵀ·dY over `rows` rows (both stored row-major → MN-major operands)
int lin_dw(cudaStream_t st, const bf16* X, int ldx, int in, const bf16* dY, int lddy, int out, long long rows,
           float* dW) {
  GemmArgs g = G_(X, ldx, 1, dY, lddy, 1, in, out, rows);
  g.flags = EPI_OUT_F32 | EPI_ATOMIC;
  g.split_k = 0;
  g.C = dW; g.ldc = out;
  return gemm_launch(g, st);
}

// Y[rows, out] (bf16) = X·W (+ bias) with W a column block of a wider row-major matrix (row stride ldw)
int lin_fwd_w(cudaStream_t st, const bf16* X, int ldx, long long rows, const bf16* W, int ldw, int in, int out,
              const float* bias, bf16* Y, int ldy) {
  GemmArgs g = G_(X, ldx, 0, W, ldw, 1, rows, out, in);
  g.flags = (bias ? EPI_BIAS : 0u) | EPI_OUT_BF16;
  g.bias = bias; g.C_bf16 = Y; g.ldc_bf = ldy;
  return gemm_launch(g, st);
}

RowMap rows_plain(const float* x, int ld, long long rows) {
  RowMap r{};
  r.A = x; r.lda = ld; r.a_rows = (int)rows; r.a_off = 0; r.na = (int)rows; r.Bsrc = nullptr; r.ldb = 0; r.nb = 0;
  r.batch = 1;
  return r;
}
RowMapW rows_plain_w(float* x, int ld, long long rows) {
  RowMapW r{};
  r.A = x; r.lda = ld; r.a_rows = (int)rows; r.a_off = 0; r.na = (int)rows; r.Bsrc = nullptr; r.ldb = 0; r.nb = 0;
  r.batch = 1;
  return r;
}

// ------------------------------------------------------------------ weight packing
void add_spec(PackList& L, long long src, void* dst, void* base, int rows, int cols, int src_ld, int dst_ld,
              int to_bf16, int dst_col = 0) {
  CopySpec s;
  const long long byte_off = reinterpret_cast<char*>(dst) - reinterpret_cast<char*>(base);
  const int esz = to_bf16 ? 2 : 4;
  s.src_off = (int)src;
  s.dst_off = (int)(byte_off / esz) + dst_col;
  s.rows = rows; s.cols = cols; s.src_ld = src_ld; s.dst_ld = dst_ld; s.to_bf16 = to_bf16;
  L.s[L.n++] = s;
}

int pack_weights(const Plan& p, const float* params, void* ws, cudaStream_t st) {
  PackList L;
  L.n = 0;
  const ParamOff& o = p.po;
  const int d = p.d, D = p.D;
  // bf16 destinations are addressed in bf16 elements from ws; fp32 in floats from ws (both 256-aligned)
  add_spec(L, o.seq_w1, p.pk.seq_w1, ws, d, 2 * D, 2 * D, 2 * D, 1);
  add_spec(L, o.seq_w2, p.pk.seq_w2, ws, 2 * D, d, d, d, 1);
  add_spec(L, o.glob_w1, p.pk.glob_w1, ws, D, 2 * D, 2 * D, 2 * D, 1);
  add_spec(L, o.glob_w2, p.pk.glob_w2, ws, 2 * D, D, D, D, 1);
  for (int i = 0; i < p.IL; ++i) {
    const BlockOff& b = o.inner[i];
    add_spec(L, b.w_q, p.pk.in_wqkv[i], ws, d, d, d, 3 * d, 1, 0);
    add_spec(L, b.w_k, p.pk.in_wqkv[i], ws, d, d, d, 3 * d, 1, d);
    add_spec(L, b.w_v, p.pk.in_wqkv[i], ws, d, d, d, 3 * d, 1, 2 * d);
    add_spec(L, b.b_q, p.pk.in_bqkv[i], ws, 1, d, d, d, 0, 0);
    add_spec(L, b.b_k, p.pk.in_bqkv[i], ws, 1, d, d, d, 0, d);
    add_spec(L, b.b_v, p.pk.in_bqkv[i], ws, 1, d, d, d, 0, 2 * d);
    add_spec(L, b.w_o, p.pk.in_wo[i], ws, d, d, d, d, 1);
    add_spec(L, b.w1, p.pk.in_w1[i], ws, d, 4 * d, 4 * d, 4 * d, 1);
    add_spec(L, b.w2, p.pk.in_w2[i], ws, 4 * d, d, d, d, 1);
  }
  {
    const BlockOff& b = o.cross;
    add_spec(L, b.w_q, p.pk.c_wq, ws, D, D, D, D, 1);
    add_spec(L, b.w_k, p.pk.c_wkv, ws, D, D, D, 2 * D, 1, 0);
    add_spec(L, b.w_v, p.pk.c_wkv, ws, D, D, D, 2 * D, 1, D);
    add_spec(L, b.b_k, p.pk.c_bkv, ws, 1, D, D, D, 0, 0);
    add_spec(L, b.b_v, p.pk.c_bkv, ws, 1, D, D, D, 0, D);
    add_spec(L, b.w_o, p.pk.c_wo, ws, D, D, D, D, 1);
    add_spec(L, b.w1, p.pk.c_w1, ws, D, 4 * D, 4 * D, 4 * D, 1);
    add_spec(L, b.w2, p.pk.c_w2, ws, 4 * D, D, D, D, 1);
  }
  for (int i = 0; i < p.N; ++i) {
    const BlockOff& b = o.self_[i];
    add_spec(L, b.w_q, p.pk.s_wqkv[i], ws, D, D, D, 3 * D, 1, 0);
    add_spec(L, b.w_k, p.pk.s_wqkv[i], ws, D, D, D, 3 * D, 1, D);
    add_spec(L, b.w_v, p.pk.s_wqkv[i], ws, D, D, D, 3 * D, 1, 2 * D);
    add_spec(L, b.b_q, p.pk.s_bqkv[i], ws, 1, D, D, D, 0, 0);
    add_spec(L, b.b_k, p.pk.s_bqkv[i], ws, 1, D, D, D, 0, D);
    add_spec(L, b.b_v, p.pk.s_bqkv[i], ws, 1, D, D, D, 0, 2 * D);
    add_spec(L, b.w_o, p.pk.s_wo[i], ws, D, D, D, D, 1);
    add_spec(L, b.w1, p.pk.s_w1[i], ws, D, 4 * D, 4 * D, 4 * D, 1);
    add_spec(L, b.w2, p.pk.s_w2[i], ws, 4 * D, D, D, D, 1);
  }
  pack_params(params, L, ws, st);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ forward
bool use_attn_tc(const AttnArgs& a) {
  return g_knobs.attn_tc && attn_tc_supported(a) != 0;
}

// One pre-norm attention block over the q query rows (pkg/src/longrec/attention.py:172-212).
// xq_src (optional): the query rows as [merged | globals] views; LN1 reads them there and
// materialises xq (the residual) itself, instead of separate gather kernels
int block_fwd(const Ctx& c, const BlockOff& bo, BlockBufs& b, const float* xq, bool cross, const bf16* Wqkv,
              const float* bqkv, const bf16* Wo, const bf16* W1, const bf16* W2, bool compact = false,
              const RowMap* xq_src = nullptr) {
  const Plan& p = c.p;
  cudaStream_t st = c.st;
  const int D = p.D;
  const long long Q = (long long)p.B * p.q;
  if (xq_src)
    layernorm_fwd(*xq_src, D, c.w(bo.ln1_g), c.w(bo.ln1_b), b.qn, b.m1, b.r1, st, const_cast<float*>(xq));
  else
    layernorm_fwd(rows_plain(xq, D, Q), D, c.w(bo.ln1_g), c.w(bo.ln1_b), b.qn, b.m1, b.r1, st);
  AttnArgs a{};
  a.nq = p.q; a.D = D; a.heads = p.heads; a.k = p.k; a.G = p.G; a.npg = p.npg; a.B = p.B;
  a.qg = (p.qs == QS_UNIFORM || p.qs == QS_RECENT_UNIFORM) ? p.qg : nullptr;
  a.learn = p.qs == QS_LEARNABLE; a.self_keys = cross ? 0 : 1;
  a.ctx = b.ctx; a.ldc = D; a.sc = (long long)p.q * D; a.lse = b.lse; a.ctx32 = b.ctx32;
  if (cross) {
    // K/V rows: LN1 + [K | V] projection were forked onto the side stream by forward()
    TRY(lin_fwd(st, b.qn, D, Q, Wqkv, D, D, c.w(bo.b_q), 0, nullptr, b.qkv, nullptr));
    if (p.absorb) {
      // S = Q·Kᵀ = (Q·W_kᵀ)·knᵀ + Q·b_k (constant per row: the softmax drops it), so the
      // attention runs on Q' = Q·W_kᵀ against the LN'd key rows kn themselves, both as keys and
      // as values: P·V = (P·kn)·W_v + b_v (rows of P sum to 1)
      TRY(lin_dx(st, b.qkv, D, Q, p.pk.c_wkv, 2 * D, D, D, nullptr, 0, p.xa_qabs, D));
    }
    join_side(st, side_stream(st));
    if (p.absorb) {
      a.Q = p.xa_qabs; a.ldq = D; a.sq = (long long)p.q * D;
      a.Kp = p.kn; a.ldk = D; a.sk = (long long)p.v * D;
      a.V = p.kn; a.ldv = D; a.sv = (long long)p.v * D;
      a.ctx = p.xa_craw; a.ctx32 = p.xa_craw32;
      a.sum_kv = 1;                                  // keys are values: one shared tile per chunk
    } else {
      a.Q = b.qkv; a.ldq = D; a.sq = (long long)p.q * D;
      a.Kp = p.KV; a.ldk = 2 * D; a.sk = (long long)p.v * 2 * D;
      a.V = p.KV + D; a.ldv = 2 * D; a.sv = (long long)p.v * 2 * D;
    }
    a.nk = p.v; a.ns = p.G; a.goff = 0;
  } else {
    TRY(lin_fwd(st, b.qn, D, Q, Wqkv, D, 3 * D, bqkv, 0, nullptr, b.qkv, nullptr));
    a.Q = b.qkv; a.ldq = 3 * D; a.sq = (long long)p.q * 3 * D;
    a.Kp = b.qkv + D; a.ldk = 3 * D; a.sk = a.sq;
    a.V = b.qkv + 2 * D; a.ldv = 3 * D; a.sv = a.sq;
    a.nk = p.q; a.ns = p.k; a.goff = p.G - p.k;
  }
  if (use_attn_tc(a)) {
    a.ctx32 = nullptr;                  // only the SIMT backward reads the fp32 context
    if (cross) probe(PH_XATTN_FWD, 0, st);
    TRY(attn_tc_fwd(a, st));
    if (cross) probe(PH_XATTN_FWD, 1, st);
  } else {
    attn_fwd(a, st);
  }
  if (cross && p.absorb)   // ctx = (P·kn)·W_v + b_v
    TRY(lin_fwd_w(st, p.xa_craw, D, Q, p.pk.c_wkv + D, 2 * D, D, D, p.pk.c_bkv + D, b.ctx, D));
  // compact: only the two rows the head reads leave the last block (model.py:346-362), so its
  // row-wise tail (W_o + residual, LN2, FFN) runs on [2B, D] gathered rows
  const long long R = compact ? 2LL * p.B : Q;
  const bf16* ctx_rows = b.ctx;
  const float* res_rows = xq;
  if (compact) {
    head_rows_gather_pair(b.ctx, p.hc_ctx, xq, p.hc_x, p.B, p.q, p.k + 1, p.k + p.m - 1, D, st);
    ctx_rows = p.hc_ctx;
    res_rows = p.hc_x;
  }
  TRY(lin_fwd(st, ctx_rows, D, R, Wo, D, D, c.w(bo.b_o), 0, b.x1, nullptr, nullptr, res_rows, D));
  layernorm_fwd(rows_plain(b.x1, D, R), D, c.w(bo.ln2_g), c.w(bo.ln2_b), b.x1n, b.m2, b.r2, st);
  TRY(lin_fwd(st, b.x1n, D, R, W1, D, 4 * D, c.w(bo.b1), EPI_GELU | EPI_SAVE_PRE, nullptr, b.gf, b.f1));
  TRY(lin_fwd(st, b.gf, 4 * D, R, W2, 4 * D, D, c.w(bo.b2), 0, b.out, nullptr, nullptr, b.x1, D));
  return 0;
}

int inner_unfused_fwd(const Ctx& c, const Plan& p);

// Featuriser + token MLP with per-stage kernels (keeps feat, x0, a1, g1 for the per-stage backward).
int mlp_unfused_fwd(const Ctx& c, const Plan& p, const LongerBatch& bt);

// Unfused front-end: featuriser kernel + tcgen05 GEMMs per stage; keeps every activation the
// unfused backward needs.
int frontend_unfused_fwd(const Ctx& c, const Plan& p, const LongerBatch& bt) {
  TRY(mlp_unfused_fwd(c, p, bt));
  return inner_unfused_fwd(c, p);
}

int mlp_unfused_fwd(const Ctx& c, const Plan& p, const LongerBatch& bt) {
  cudaStream_t st = c.st;
  const ParamOff& o = p.po;
  const LongerDims& dm = p.dims;
  const int d = p.d, D = p.D;
  const long long T = p.T;
  // featurise + recency position (inputs.py:434-482)
  EmbedArgs e{};
  e.items = bt.items; e.actions = bt.actions; e.dt = bt.dt; e.n_events = bt.n_events;
  e.B = p.B; e.L = p.L; e.Lp = p.Lp; e.d = d; e.d_item = dm.d_item; e.d_act = dm.d_act; e.d_time = dm.d_time;
  e.FP = p.FP; e.nb = dm.n_time_buckets; e.vocab = dm.vocab; e.n_actions = dm.n_actions; e.K = p.K;
  e.item_tab = c.w(o.item); e.act_tab = c.w(o.act); e.time_tab = c.w(o.time); e.pos_tab = c.w(o.pos);
  e.tok_w = c.w(o.tok_w); e.tok_b = c.w(o.tok_b);
  e.feat = p.feat; e.x0 = p.x0; e.real = p.real; e.keep = p.keep; e.status = p.status; e.npg = p.npg;
  embed_fwd(e, st);
  // per-token input MLP (inputs.py:447-449); pad rows zeroed (inputs.py:478-481)
  TRY(lin_fwd(st, p.x0, d, T, p.pk.seq_w1, d, 2 * D, c.w(o.seq_b1), EPI_GELU | EPI_SAVE_PRE, nullptr, p.g1, p.a1));
  TRY(lin_fwd(st, p.g1, 2 * D, T, p.pk.seq_w2, 2 * D, d, c.w(o.seq_b2), 0, p.h, nullptr, nullptr, nullptr, 0, p.real));
  return 0;
}

// InnerTrans merge (merge.py:83-112) from p.h with per-stage kernels, keeping every activation
// the per-stage backward needs.  With the fused front-end this is the backward's recompute.
int inner_unfused_fwd(const Ctx& c, const Plan& p) {
  cudaStream_t st = c.st;
  const ParamOff& o = p.po;
  const int d = p.d;
  const long long T = p.T;
  const float* x = p.h;
  for (int i = 0; i < p.IL; ++i) {
    const InnerBufs& b = p.in[i];
    const BlockOff& bo = o.inner[i];
    layernorm_fwd(rows_plain(x, d, T), d, c.w(bo.ln1_g), c.w(bo.ln1_b), b.xn, b.m1, b.r1, st);
    TRY(lin_fwd(st, b.xn, d, T, p.pk.in_wqkv[i], d, 3 * d, p.pk.in_bqkv[i], 0, b.qkv, nullptr, nullptr));
    group_attn_fwd(b.qkv, (int)T, p.K, d, b.ctx, b.probs, st);
    TRY(lin_fwd(st, b.ctx, d, T, p.pk.in_wo[i], d, d, c.w(bo.b_o), 0, b.x1, nullptr, nullptr, x, d));
    layernorm_fwd(rows_plain(b.x1, d, T), d, c.w(bo.ln2_g), c.w(bo.ln2_b), b.x1n, b.m2, b.r2, st);
    TRY(lin_fwd(st, b.x1n, d, T, p.pk.in_w1[i], d, 4 * d, c.w(bo.b1), EPI_GELU | EPI_SAVE_PRE, nullptr, b.gf, b.f1));
    TRY(lin_fwd(st, b.gf, 4 * d, T, p.pk.in_w2[i], 4 * d, d, c.w(bo.b2), 0, b.out, nullptr, nullptr, b.x1, d,
                i == p.IL - 1 ? p.keep : nullptr));
    x = b.out;
  }
  return 0;
}

FrontArgs front_args(const Ctx& c, const Plan& p, const LongerBatch& bt) {
  const ParamOff& o = p.po;
  const LongerDims& dm = p.dims;
  FrontArgs f{};
  f.items = bt.items; f.actions = bt.actions; f.dt = bt.dt; f.n_events = bt.n_events;
  f.B = p.B; f.L = p.L; f.Lp = p.Lp; f.K = p.K; f.d = p.d; f.d_item = dm.d_item; f.d_act = dm.d_act;
  f.d_time = dm.d_time; f.nb = dm.n_time_buckets; f.vocab = dm.vocab; f.n_actions = dm.n_actions;
  f.inner_layers = p.IL; f.T = p.T;
  f.item_tab = c.w(o.item); f.act_tab = c.w(o.act); f.time_tab = c.w(o.time); f.pos_tab = c.w(o.pos);
  f.tok_w = c.w(o.tok_w); f.tok_b = c.w(o.tok_b); f.seq_b1 = c.w(o.seq_b1); f.seq_b2 = c.w(o.seq_b2);
  for (int l = 0; l < p.IL; ++l) {
    const BlockOff& b = o.inner[l];
    f.inner_bias[l][0] = c.w(b.b_q); f.inner_bias[l][1] = c.w(b.b_k); f.inner_bias[l][2] = c.w(b.b_v);
    f.inner_bias[l][3] = c.w(b.b_o); f.inner_bias[l][4] = c.w(b.b1); f.inner_bias[l][5] = c.w(b.b2);
    f.inner_ln[l][0] = c.w(b.ln1_g); f.inner_ln[l][1] = c.w(b.ln1_b);
    f.inner_ln[l][2] = c.w(b.ln2_g); f.inner_ln[l][3] = c.w(b.ln2_b);
  }
  f.wblob = p.wblob;
  f.proj = p.proj;
  f.merged = p.merged; f.status = p.status; f.npg = p.npg;
  f.h_out = p.IL ? p.h : nullptr;
  f.real_out = p.real; f.keep_out = p.keep;
  if (c.G) {
    f.g_tok_w = c.g(o.tok_w); f.g_tok_b = c.g(o.tok_b); f.g_seq_w1 = c.g(o.seq_w1); f.g_seq_b1 = c.g(o.seq_b1);
    f.g_seq_w2 = c.g(o.seq_w2); f.g_seq_b2 = c.g(o.seq_b2); f.g_item = c.g(o.item); f.g_act = c.g(o.act);
    f.g_time = c.g(o.time); f.g_pos = c.g(o.pos);
  }
  return f;
}

// Fused front-end (frontend.cu): ids → merged rows in one persistent kernel.
int frontend_fused_fwd(const Ctx& c, const Plan& p, const LongerBatch& bt) {
  const ParamOff& o = p.po;
  long long iw[kMaxInner][4];
  for (int l = 0; l < p.IL; ++l) {
    iw[l][0] = o.inner[l].w_q; iw[l][1] = o.inner[l].w_k; iw[l][2] = o.inner[l].w_v; iw[l][3] = o.inner[l].w_o;
  }
  const LongerDims& dm = p.dims;
  const ProjArgs pj{c.w(o.item), c.w(o.act), c.w(o.time), c.w(o.tok_w), c.w(o.tok_b), dm.vocab, dm.n_actions,
                    dm.n_time_buckets, dm.d_item, dm.d_act, dm.d_time, p.d, p.proj};
  pack_frontend_weights(c.P, o.tok_w, o.seq_w1, o.seq_w2, iw, p.d, p.D, p.F, p.IL, p.wblob, pj, c.st);
  FrontArgs f = front_args(c, p, bt);
  // epilogue: the cross block's LN1 of the merged rows straight into the K/V operand (kn)
  f.kn = p.kn; f.kn_g = c.w(o.cross.ln1_g); f.kn_b = c.w(o.cross.ln1_b);
  f.kn_mean = p.mk; f.kn_rstd = p.rk; f.v = p.v;
  return frontend_fwd(f, c.st);
}

// O = [merged[G-k:]; globals] per sample (the "recent" strategy) as a RowMap over the two sources
RowMap recent_query_rows(const Plan& p) {
  RowMap r{};
  r.A = p.merged; r.lda = p.D; r.a_rows = p.G; r.a_off = p.G - p.k; r.na = p.k;
  r.Bsrc = p.glob; r.ldb = p.D; r.nb = p.m; r.batch = p.B;
  return r;
}

int forward(const Ctx& c, const Plan& p, const LongerBatch& bt, float* probs, float* loss, int with_loss) {
  cudaStream_t st = c.st;
  const ParamOff& o = p.po;
  const LongerDims& dm = p.dims;
  const int d = p.d, D = p.D;
  const long long M = (long long)p.B * p.m;
  (void)with_loss;
  // global tokens (inputs.py:500-537): independent of the sequence front-end, so they run on the
  // side stream beside it; main waits for them only where the query rows take the globals.  With
  // the fused front-end (its own weight blob) the bf16 GEMM operand copies are packed there too:
  // the main stream first needs them after that wait.
  const cudaStream_t ss = side_stream(st);
  if (!p.fused_fe) TRY(pack_weights(p, c.P, p.ws, st));
  fork_side(st, ss);
  if (p.fused_fe) TRY(pack_weights(p, c.P, p.ws, ss));
  GlobalsArgs ga{};
  ga.uid = bt.uid; ga.cand_item = bt.cand_item; ga.B = p.B; ga.m = p.m; ga.d = d; ga.D = D;
  ga.d_item = dm.d_item; ga.d_act = dm.d_act; ga.d_time = dm.d_time;
  ga.uid_tab = c.w(o.uid); ga.item_tab = c.w(o.item); ga.time_tab = c.w(o.time); ga.cls = c.w(o.cls);
  ga.tok_w = c.w(o.tok_w); ga.tok_b = c.w(o.tok_b); ga.lift_w = c.w(o.lift_w); ga.lift_b = c.w(o.lift_b);
  ga.raw = p.raw; ga.raw_bf = p.raw_bf; ga.td = p.td;
  globals_raw_fwd(ga, ss);
  TRY(lin_fwd(ss, p.raw_bf, D, M, p.pk.glob_w1, D, 2 * D, c.w(o.glob_b1), EPI_GELU | EPI_SAVE_PRE, nullptr, p.gg, p.ga));
  TRY(lin_fwd(ss, p.gg, 2 * D, M, p.pk.glob_w2, 2 * D, D, c.w(o.glob_b2), 0, p.glob, nullptr, nullptr));
  mark_side(st, ss);
  if (p.fused_fe) {
    probe(PH_FE_FWD, 0, c.st); TRY(frontend_fused_fwd(c, p, bt)); probe(PH_FE_FWD, 1, c.st);
    probe(PH_FWD_ROWS, 0, c.st);
  } else {
    TRY(frontend_unfused_fwd(c, p, bt));
  }
  // composite queries O = [merged[G-k:]; globals] (model.py:317-319)
  {
    // R = [merged; globals] → cross LN1 → [K | V] over all B·v rows, on the side stream (after the
    // globals) while the main stream builds the q query rows (joined in block_fwd before the attention)
    fork_side(st, ss);
    RowMap r{};
    if (p.fused_fe) {          // merged rows were normalised by the fused front-end; globals only
      r.A = p.glob; r.lda = D; r.a_rows = p.m; r.a_off = 0; r.na = p.m; r.Bsrc = nullptr; r.ldb = D; r.nb = 0;
      r.o_per = p.v; r.o_off = p.G;
    } else {
      r.A = p.merged; r.lda = D; r.a_rows = p.G; r.a_off = 0; r.na = p.G; r.Bsrc = p.glob; r.ldb = D; r.nb = p.m;
    }
    r.batch = p.B;
    layernorm_fwd(r, D, c.w(o.cross.ln1_g), c.w(o.cross.ln1_b), p.kn, p.mk, p.rk, ss);
    if (!p.absorb)
      TRY(lin_fwd(ss, p.kn, D, (long long)p.B * p.v, p.pk.c_wkv, D, 2 * D, p.pk.c_bkv, 0, nullptr, p.KV, nullptr));
  }
  // sequence queries (select_queries, model.py:58-123).  "recent" queries are the last k merged
  // rows: the cross block's LN1 reads them (and the globals) in place and materialises O itself
  const RowMap qrows = recent_query_rows(p);
  if (p.qs != QS_RECENT) {
    if (p.qs != QS_LEARNABLE) select_queries(p.npg, p.B, p.G, p.k, p.qs, p.qg, st);
    gather_query_rows(p.merged, p.qs == QS_LEARNABLE ? nullptr : p.qg, p.qs == QS_LEARNABLE ? c.w(o.qbank) : nullptr,
                      p.B, p.G, p.k, D, p.O, p.q, st);
  }
  wait_mark(st, ss);                                   // the global rows
  if (p.qs != QS_RECENT) gather_rows_f32(p.glob, p.B, p.m, 0, p.m, p.O, p.q, p.k, D, st);
  Plan& pm = const_cast<Plan&>(p);
  TRY(block_fwd(c, o.cross, pm.cb, p.O, true, p.pk.c_wq, nullptr, p.pk.c_wo, p.pk.c_w1, p.pk.c_w2, false,
                p.qs == QS_RECENT ? &qrows : nullptr));
  const float* xl = p.cb.out;
  for (int i = 0; i < p.N; ++i) {
    TRY(block_fwd(c, o.self_[i], pm.sb[i], xl, false, p.pk.s_wqkv[i], p.pk.s_bqkv[i], p.pk.s_wo[i], p.pk.s_w1[i],
                  p.pk.s_w2[i], p.compact_head && i == p.N - 1));
    xl = p.sb[i].out;
  }
  HeadArgs h{};
  h.x = xl; h.B = p.B; h.q = p.q; h.k = p.k; h.m = p.m; h.D = D; h.d = d; h.hh = p.hh;
  if (p.compact_head) { h.q = 2; h.k = -1; h.m = 3; }   // rows k+1, k+m−1 → compact rows 0, 1
  h.uid = bt.uid; h.profile = bt.profile; h.label = bt.label;
  h.uid_tab = c.w(o.uid); h.prof_tab = c.w(o.prof);
  h.w1 = c.w(o.head_w1); h.b1 = c.w(o.head_b1); h.w2 = c.w(o.head_w2); h.b2 = c.w(o.head_b2);
  h.hin = p.hin; h.z1 = p.z1; h.probs = probs;
  h.loss_per = with_loss ? p.loss_per : nullptr; h.dz = p.dz; h.loss = loss;
  head_fwd(h, 0, st);
  if (with_loss) {          // the scalar loss feeds nothing on the device: off the critical chain
    fork_side(st, ss);
    loss_mean(p.loss_per, p.B, loss, ss);
    if (!c.G) join_side(st, ss);   // forward-only call: joined before return
  }
  if (p.fused_fe) probe(PH_FWD_ROWS, 1, st);
  TRY((int)cudaGetLastError());
  return 0;
}

// Backward of one attention block (pkg/src/longrec/attention.py:172-212 + tensors.py backward
// closures).  dL/d(out) is in b.g_dx (fp32) / b.g_dx_bf (bf16).  The critical dX chain runs on
// c.st; every weight gradient and bias column sum goes to the side stream ss.
//   self:  dL/d(x_q) → nxt_dx / nxt_dx_bf (the previous block's g_dx), with the column sums of it
//          accumulated into nxt_b2 (that block's FFN output bias gradient).
//   cross: dL/d(merged rows) → p.dmerged, dL/d(global rows) → p.dglob.
int block_bwd(const Ctx& c, cudaStream_t ss, const BlockOff& bo, const BlockBufs& b, const float* xq, bool cross,
              const bf16* Wqkv, const bf16* Wo, const bf16* W1, const bf16* W2, float* nxt_dx, bf16* nxt_dx_bf,
              float* nxt_b2, bool compact = false) {
  const Plan& p = c.p;
  cudaStream_t st = c.st;
  const int D = p.D;
  const long long Q = (long long)p.B * p.q, V = (long long)p.B * p.v;
  // FFN + residual (compact: the last block's tail ran on the two head rows per sample)
  const long long R = compact ? 2LL * p.B : Q;
  float* dx1_rows = compact ? p.hc_g : b.g_dx1;
  bf16* dx1_bf_rows = compact ? p.hc_g_bf : b.g_dx1_bf;
  fork_side(st, ss);
  TRY(lin_dw(ss, b.gf, 4 * D, 4 * D, b.g_dx_bf, D, D, R, c.g(bo.w2)));
  TRY(lin_dx(st, b.g_dx_bf, D, R, W2, D, 4 * D, D, nullptr, 0, b.g_df1, 4 * D, b.f1));
  fork_side(st, ss);
  TRY(lin_dw(ss, b.x1n, D, D, b.g_df1, 4 * D, 4 * D, R, c.g(bo.w1)));
  colsum_bf16(b.g_df1, (int)R, 4 * D, 4 * D, c.g(bo.b1), ss);
  TRY(lin_dx(st, b.g_df1, 4 * D, R, W1, 4 * D, D, 4 * D, b.g_dx1n, D, nullptr, 0));
  {
    LnBwdExtra ex;
    ex.addend = b.g_dx; ex.out_bf = dx1_bf_rows; ex.colsum_out = c.g(bo.b_o);
    layernorm_bwd(rows_plain(b.x1, D, R), D, c.w(bo.ln2_g), b.m2, b.r2, b.g_dx1n, D, rows_plain_w(dx1_rows, D, R), 0,
                  nullptr, c.g(bo.ln2_g), c.g(bo.ln2_b), st, ex);
  }
  // output projection
  fork_side(st, ss);
  TRY(lin_dw(ss, compact ? p.hc_ctx : b.ctx, D, D, dx1_bf_rows, D, D, R, c.g(bo.w_o)));
  const bool absorb = cross && p.absorb;
  TRY(lin_dx(st, dx1_bf_rows, D, R, Wo, D, D, D, compact ? p.hc_dctx : b.g_dctx, D, absorb ? p.xa_dctx_bf : nullptr,
             D));
  if (compact) {   // back to full [B·q, D] rows (zero elsewhere) for the attention and LN1 backward
    head_rows_scatter_pair(p.hc_dctx, b.g_dctx, p.hc_g, b.g_dx1, p.B, p.q, p.k + 1, p.k + p.m - 1, D, st);
  }
  // attention
  AttnArgs a{};
  a.nq = p.q; a.D = D; a.heads = p.heads; a.k = p.k; a.G = p.G; a.npg = p.npg; a.B = p.B;
  a.qg = (p.qs == QS_UNIFORM || p.qs == QS_RECENT_UNIFORM) ? p.qg : nullptr;
  a.learn = p.qs == QS_LEARNABLE; a.self_keys = cross ? 0 : 1;
  a.ctx = b.ctx; a.ldc = D; a.sc = (long long)p.q * D; a.lse = b.lse; a.ctx32 = b.ctx32;
  a.dctx = b.g_dctx; a.lddc = D; a.sdc = (long long)p.q * D; a.ctx_in = b.ctx;
  if (absorb) {
    // ctx = C·W_v + b_v with C = P·kn: dW_v = Cᵀ·dctx, db_v = Σ dctx (side stream), dC = dctx·W_vᵀ;
    // the attention backward then runs on (Q', kn, kn) with dO = dC: dQ', and dK + dV summed
    // straight into d(kn) (the K / V rows are kn itself)
    fork_side(st, ss);
    TRY(lin_dw(ss, p.xa_craw, D, D, p.xa_dctx_bf, D, D, Q, c.g(bo.w_v)));
    colsum_f32(b.g_dctx, (int)Q, D, D, c.g(bo.b_v), ss);
    TRY(lin_dx(st, p.xa_dctx_bf, D, Q, p.pk.c_wkv + D, 2 * D, D, D, p.xa_dC, D, nullptr, 0));
    a.ctx = p.xa_craw; a.ctx32 = p.xa_craw32; a.ctx_in = p.xa_craw;
    a.dctx = p.xa_dC;
    a.Q = p.xa_qabs; a.ldq = D; a.sq = (long long)p.q * D;
    a.Kp = p.kn; a.ldk = D; a.sk = (long long)p.v * D;
    a.V = p.kn; a.ldv = D; a.sv = a.sk;
    a.nk = p.v; a.ns = p.G; a.goff = 0;
    a.dQ = p.xa_dqabs; a.lddq = D; a.sdq = (long long)p.q * D;
    bf16* dkn_bf = reinterpret_cast<bf16*>(p.dkn);
    a.dK = dkn_bf; a.lddk = D; a.sdk = (long long)p.v * D;
    a.dV = dkn_bf; a.lddv = D; a.sdv = a.sdk;
    a.sum_kv = 1;
  } else if (cross) {
    a.Q = b.qkv; a.ldq = D; a.sq = (long long)p.q * D;
    a.Kp = p.KV; a.ldk = 2 * D; a.sk = (long long)p.v * 2 * D;
    a.V = p.KV + D; a.ldv = 2 * D; a.sv = a.sk;
    a.nk = p.v; a.ns = p.G; a.goff = 0;
    a.dQ = b.g_dqkv; a.lddq = D; a.sdq = (long long)p.q * D;
    a.dK = p.dKV; a.lddk = 2 * D; a.sdk = (long long)p.v * 2 * D;
    a.dV = p.dKV + D; a.lddv = 2 * D; a.sdv = a.sdk;
  } else {
    a.Q = b.qkv; a.ldq = 3 * D; a.sq = (long long)p.q * 3 * D;
    a.Kp = b.qkv + D; a.ldk = 3 * D; a.sk = a.sq;
    a.V = b.qkv + 2 * D; a.ldv = 3 * D; a.sv = a.sq;
    a.nk = p.q; a.ns = p.k; a.goff = p.G - p.k;
    a.dQ = b.g_dqkv; a.lddq = 3 * D; a.sdq = (long long)p.q * 3 * D;
    a.dK = b.g_dqkv + D; a.lddk = 3 * D; a.sdk = a.sdq;
    a.dV = b.g_dqkv + 2 * D; a.lddv = 3 * D; a.sdv = a.sdq;
  }
  if (use_attn_tc(a)) {
    if (cross) probe(PH_XATTN_BWD, 0, st);
    TRY(attn_tc_bwd(a, st));
    if (cross) probe(PH_XATTN_BWD, 1, st);
  } else {
    attn_bwd(a, st);
  }
  // absorbed: dQ = dQ'·W_k, dW_k = dQ'ᵀ·Q (S = Q·W_kᵀ·knᵀ); b_k's gradient is exactly 0 (the
  // softmax is invariant to it) and stays so
  if (absorb) TRY(lin_fwd_w(st, p.xa_dqabs, D, Q, p.pk.c_wkv, 2 * D, D, D, nullptr, b.g_dqkv, D));
  fork_side(st, ss);
  if (cross) {
    TRY(lin_dw(ss, b.qn, D, D, b.g_dqkv, D, D, Q, c.g(bo.w_q)));
    colsum_bf16(b.g_dqkv, (int)Q, D, D, c.g(bo.b_q), ss);
    bf16* dkn_bf = reinterpret_cast<bf16*>(p.dkn);
    if (absorb) {
      TRY(lin_dw(ss, p.xa_dqabs, D, D, b.qkv, D, D, Q, c.g(bo.w_k)));
    } else {
      TRY(lin_dw(ss, p.kn, D, D, p.dKV, 2 * D, D, V, c.g(bo.w_k)));
      TRY(lin_dw(ss, p.kn, D, D, p.dKV + D, 2 * D, D, V, c.g(bo.w_v)));
      colsum_bf16(p.dKV, (int)V, D, 2 * D, c.g(bo.b_k), ss);
      colsum_bf16(p.dKV + D, (int)V, D, 2 * D, c.g(bo.b_v), ss);
    }
    TRY(lin_dx(st, b.g_dqkv, D, Q, Wqkv, D, D, D, b.g_dqn, D, nullptr, 0));
    // dK|dV → d(kn) in bf16 (it only feeds the HBM-bound LN backward below), in p.dkn's storage
    if (!absorb) TRY(lin_dx(st, p.dKV, 2 * D, V, p.pk.c_wkv, 2 * D, D, 2 * D, nullptr, 0, dkn_bf, D));
    RowMap r{};
    r.A = p.merged; r.lda = D; r.a_rows = p.G; r.a_off = 0; r.na = p.G; r.Bsrc = p.glob; r.ldb = D; r.nb = p.m;
    r.batch = p.B;
    RowMapW rw{};
    rw.A = p.dmerged; rw.lda = D; rw.a_rows = p.G; rw.a_off = 0; rw.na = p.G; rw.Bsrc = p.dglob; rw.ldb = D;
    rw.nb = p.m; rw.batch = p.B;
    layernorm_bwd(r, D, c.w(bo.ln1_g), p.mk, p.rk, dkn_bf, D, rw, c.g(bo.ln1_g), c.g(bo.ln1_b), st);
    LnBwdExtra ex;
    ex.addend = b.g_dx1;
    if (p.qs == QS_RECENT) {
      // straight into the query rows' sources: += into dmerged[G-k:] and dglob (which the K/V-row
      // LN backward above has just written)
      RowMapW qw{};
      qw.A = p.dmerged; qw.lda = D; qw.a_rows = p.G; qw.a_off = p.G - p.k; qw.na = p.k;
      qw.Bsrc = p.dglob; qw.ldb = D; qw.nb = p.m; qw.batch = p.B;
      layernorm_bwd(recent_query_rows(p), D, c.w(bo.ln1_g), b.m1, b.r1, b.g_dqn, D, qw, 1, nullptr,
                    c.g(bo.ln1_g), c.g(bo.ln1_b), st, ex);
    } else {
      layernorm_bwd(rows_plain(xq, D, Q), D, c.w(bo.ln1_g), b.m1, b.r1, b.g_dqn, D, rows_plain_w(p.dO, D, Q), 0,
                    nullptr, c.g(bo.ln1_g), c.g(bo.ln1_b), st, ex);
      scatter_query_rows(p.dO, p.q, p.qg, p.B, p.G, p.k, D, p.dmerged,
                         p.qs == QS_LEARNABLE ? c.g(p.po.qbank) : nullptr, st);
      add_rows_f32(p.dO, p.B, p.q, p.k, p.m, p.dglob, p.m, 0, D, st);
    }
  } else {
    for (int j = 0; j < 3; ++j) {
      const long long wo = j == 0 ? bo.w_q : (j == 1 ? bo.w_k : bo.w_v);
      const long long bb = j == 0 ? bo.b_q : (j == 1 ? bo.b_k : bo.b_v);
      TRY(lin_dw(ss, b.qn, D, D, b.g_dqkv + j * D, 3 * D, D, Q, c.g(wo)));
      colsum_bf16(b.g_dqkv + j * D, (int)Q, D, 3 * D, c.g(bb), ss);
    }
    TRY(lin_dx(st, b.g_dqkv, 3 * D, Q, Wqkv, 3 * D, D, 3 * D, b.g_dqn, D, nullptr, 0));
    LnBwdExtra ex;
    ex.addend = b.g_dx1; ex.out_bf = nxt_dx_bf; ex.colsum_out = nxt_b2;
    layernorm_bwd(rows_plain(xq, D, Q), D, c.w(bo.ln1_g), b.m1, b.r1, b.g_dqn, D, rows_plain_w(nxt_dx, D, Q), 0,
                  nullptr, c.g(bo.ln1_g), c.g(bo.ln1_b), st, ex);
  }
  return 0;
}

int backward(const Ctx& c, const Plan& p, const LongerBatch& bt, float* probs) {
  cudaStream_t st = c.st;
  const ParamOff& o = p.po;
  const LongerDims& dm = p.dims;
  const int d = p.d, D = p.D;
  const long long T = p.T, M = (long long)p.B * p.m, Q = (long long)p.B * p.q;
  const cudaStream_t ss = side_stream(st);
  const BlockBufs& last = p.N ? p.sb[p.N - 1] : p.cb;
  probe(PH_BWD_ROWS, 0, st);
  TRY((int)cudaMemsetAsync(c.G, 0, o.total * 4, st));
  TRY((int)cudaMemsetAsync(last.g_dx, 0, Q * D * 4, st));
  TRY((int)cudaMemsetAsync(last.g_dx_bf, 0, Q * D * 2, st));
  // head (model.py:346-362) → dx rows k+m-1 (target) and k+1 (CLS)
  HeadArgs h{};
  h.x = p.N ? p.sb[p.N - 1].out : p.cb.out;
  h.B = p.B; h.q = p.q; h.k = p.k; h.m = p.m; h.D = D; h.d = d; h.hh = p.hh;
  if (p.compact_head) { h.q = 2; h.k = -1; h.m = 3; }
  h.uid = bt.uid; h.profile = bt.profile; h.label = bt.label;
  h.uid_tab = c.w(o.uid); h.prof_tab = c.w(o.prof);
  h.w1 = c.w(o.head_w1); h.b1 = c.w(o.head_b1); h.w2 = c.w(o.head_w2); h.b2 = c.w(o.head_b2);
  h.hin = p.hin; h.z1 = p.z1; h.probs = probs; h.dz = p.dz; h.dz1 = p.dz1; h.dx = last.g_dx; h.dx_bf = last.g_dx_bf;
  h.g_w1 = c.g(o.head_w1); h.g_b1 = c.g(o.head_b1); h.g_w2 = c.g(o.head_w2); h.g_b2 = c.g(o.head_b2);
  h.g_uid = c.g(o.uid); h.g_prof = c.g(o.prof);
  head_bwd(h, st);
  fork_side(st, ss);
  head_wgrad(h, ss);                 // weight / table gradients: off the critical chain
  colsum_f32(last.g_dx, (int)(p.compact_head ? 2LL * p.B : Q), D, D, c.g(p.N ? o.self_[p.N - 1].b2 : o.cross.b2), ss);
  for (int i = p.N - 1; i >= 0; --i) {
    const float* xin = i == 0 ? p.cb.out : p.sb[i - 1].out;
    const BlockBufs& nb = i == 0 ? p.cb : p.sb[i - 1];
    TRY(block_bwd(c, ss, o.self_[i], p.sb[i], xin, false, p.pk.s_wqkv[i], p.pk.s_wo[i], p.pk.s_w1[i], p.pk.s_w2[i],
                  nb.g_dx, nb.g_dx_bf, c.g(i == 0 ? o.cross.b2 : o.self_[i - 1].b2), p.compact_head && i == p.N - 1));
  }
  TRY(block_bwd(c, ss, o.cross, p.cb, p.O, true, p.pk.c_wq, p.pk.c_wo, p.pk.c_w1, p.pk.c_w2, nullptr, nullptr,
                nullptr));
  if (g_grad_event) {
    // grads[cross, total) (blocks, query bank, head) are final once the side stream has also
    // drained their weight gradients: record there, after it joins main, so main never waits
    const cudaStream_t es = ss == st ? st : ss;
    fork_side(st, ss);
    record_event(g_grad_event, es);
  }
  // global-token MLP and raw rows: nothing on the token side needs them, so with the knob the
  // whole chain runs on the side stream, launched ahead of the fused token backward
  const cudaStream_t gs = g_knobs.glob_side ? ss : st;
  if (gs != st) fork_side(st, ss);
  cast_rows_bf16(p.dglob, (int)M, D, D, p.dglob_bf, D, nullptr, gs);
  if (gs == st) fork_side(st, ss);
  TRY(lin_dw(ss, p.gg, 2 * D, 2 * D, p.dglob_bf, D, D, M, c.g(o.glob_w2)));
  colsum_f32(p.dglob, (int)M, D, D, c.g(o.glob_b2), ss);
  TRY(lin_dx(gs, p.dglob_bf, D, M, p.pk.glob_w2, D, 2 * D, D, nullptr, 0, p.dga, 2 * D, p.ga));
  if (gs == st) fork_side(st, ss);
  TRY(lin_dw(ss, p.raw_bf, D, D, p.dga, 2 * D, 2 * D, M, c.g(o.glob_w1)));
  colsum_bf16(p.dga, (int)M, 2 * D, 2 * D, c.g(o.glob_b1), ss);
  TRY(lin_dx(gs, p.dga, 2 * D, M, p.pk.glob_w1, 2 * D, D, 2 * D, p.draw, D, nullptr, 0));
  GlobalsArgs ga{};
  ga.uid = bt.uid; ga.cand_item = bt.cand_item; ga.B = p.B; ga.m = p.m; ga.d = d; ga.D = D;
  ga.d_item = dm.d_item; ga.d_act = dm.d_act; ga.d_time = dm.d_time;
  ga.uid_tab = c.w(o.uid); ga.item_tab = c.w(o.item); ga.time_tab = c.w(o.time); ga.cls = c.w(o.cls);
  ga.tok_w = c.w(o.tok_w); ga.tok_b = c.w(o.tok_b); ga.lift_w = c.w(o.lift_w); ga.lift_b = c.w(o.lift_b);
  ga.td = p.td; ga.draw = p.draw;
  ga.g_uid = c.g(o.uid); ga.g_item = c.g(o.item); ga.g_time = c.g(o.time); ga.g_cls = c.g(o.cls);
  ga.g_tok_w = c.g(o.tok_w); ga.g_tok_b = c.g(o.tok_b); ga.g_lift_w = c.g(o.lift_w); ga.g_lift_b = c.g(o.lift_b);
  globals_raw_bwd(ga, gs);
  // InnerTrans backward (all-pad groups were zeroed after the last layer).  The fused forward
  // kept only its input h, so the per-stage activations are recomputed here first.
  float* dxt = p.dmerged;
  int first_unfused = p.IL - 1;
  probe(PH_BWD_ROWS, 1, st);
  if (p.fused_fe && p.IL == 1) {
    FrontArgs f = front_args(c, p, bt);
    f.h_in = p.h; f.dmerged = p.dmerged; f.dh_out = p.t_dx;
    // the fused MLP backward takes dh as a bf16 MMA operand: hand it over in bf16 (half the bytes)
    if (frontend_mlp_bwd_supported(p.d, p.K, p.D)) { f.dh_out = nullptr; f.dh_out_bf = reinterpret_cast<bf16*>(p.t_dx); }
    const BlockOff& bo = o.inner[0];
    const long long offs[16] = {bo.w_q, bo.b_q, bo.w_k, bo.b_k, bo.w_v, bo.b_v, bo.w_o, bo.b_o,
                                bo.w1, bo.b1, bo.w2, bo.b2, bo.ln1_g, bo.ln1_b, bo.ln2_g, bo.ln2_b};
    for (int i = 0; i < 16; ++i) f.g_inner[i] = c.g(offs[i]);
    probe(PH_FE_INNER_BWD, 0, st); TRY(frontend_inner_bwd(f, st)); probe(PH_FE_INNER_BWD, 1, st);
    dxt = p.t_dx;
    first_unfused = -1;
  } else if (p.fused_fe && p.IL) {
    TRY(inner_unfused_fwd(c, p));
  }
  if (first_unfused >= 0) mul_rows_inplace(dxt, (int)T, d, p.keep, st);
  for (int i = first_unfused; i >= 0; --i) {
    const InnerBufs& b = p.in[i];
    const BlockOff& bo = o.inner[i];
    const float* xin = i == 0 ? p.h : p.in[i - 1].out;
    cast_rows_bf16(dxt, (int)T, d, d, p.t_dx_bf, d, nullptr, st);
    TRY(lin_dx(st, p.t_dx_bf, d, T, p.pk.in_w2[i], d, 4 * d, d, nullptr, 0, p.t_df1, 4 * d, b.f1));
    TRY(lin_dw(st, b.gf, 4 * d, 4 * d, p.t_dx_bf, d, d, T, c.g(bo.w2)));
    colsum_f32(dxt, (int)T, d, d, c.g(bo.b2), st);
    TRY(lin_dx(st, p.t_df1, 4 * d, T, p.pk.in_w1[i], 4 * d, d, 4 * d, p.t_dx1n, d, nullptr, 0));
    TRY(lin_dw(st, b.x1n, d, d, p.t_df1, 4 * d, 4 * d, T, c.g(bo.w1)));
    colsum_bf16(p.t_df1, (int)T, 4 * d, 4 * d, c.g(bo.b1), st);
    TRY((int)cudaMemcpyAsync(p.t_dx1, dxt, T * d * 4, cudaMemcpyDeviceToDevice, st));
    layernorm_bwd(rows_plain(b.x1, d, T), d, c.w(bo.ln2_g), b.m2, b.r2, p.t_dx1n, d, rows_plain_w(p.t_dx1, d, T), 1,
                  nullptr, c.g(bo.ln2_g), c.g(bo.ln2_b), st);
    cast_rows_bf16(p.t_dx1, (int)T, d, d, p.t_dx1_bf, d, nullptr, st);
    TRY(lin_dx(st, p.t_dx1_bf, d, T, p.pk.in_wo[i], d, d, d, p.t_dctx, d, nullptr, 0));
    TRY(lin_dw(st, b.ctx, d, d, p.t_dx1_bf, d, d, T, c.g(bo.w_o)));
    colsum_f32(p.t_dx1, (int)T, d, d, c.g(bo.b_o), st);
    group_attn_bwd(b.qkv, b.probs, p.t_dctx, (int)T, p.K, d, p.t_dqkv, st);
    TRY(lin_dx(st, p.t_dqkv, 3 * d, T, p.pk.in_wqkv[i], 3 * d, d, 3 * d, p.t_dxn, d, nullptr, 0));
    for (int j = 0; j < 3; ++j) {
      const long long wo = j == 0 ? bo.w_q : (j == 1 ? bo.w_k : bo.w_v);
      const long long bb = j == 0 ? bo.b_q : (j == 1 ? bo.b_k : bo.b_v);
      TRY(lin_dw(st, b.xn, d, d, p.t_dqkv + j * d, 3 * d, d, T, c.g(wo)));
      colsum_bf16(p.t_dqkv + j * d, (int)T, d, 3 * d, c.g(bb), st);
    }
    TRY((int)cudaMemcpyAsync(p.t_dx, p.t_dx1, T * d * 4, cudaMemcpyDeviceToDevice, st));
    layernorm_bwd(rows_plain(xin, d, T), d, c.w(bo.ln1_g), b.m1, b.r1, p.t_dxn, d, rows_plain_w(p.t_dx, d, T), 1,
                  nullptr, c.g(bo.ln1_g), c.g(bo.ln1_b), st);
    dxt = p.t_dx;
  }
  // token MLP + featuriser (inputs.py:434-482); only real tokens carry gradient
  if (p.fused_fe && !frontend_mlp_bwd_supported(p.d, p.K, p.D)) {
    // widths the fused MLP backward does not take: recompute the MLP activations per stage
    TRY(mlp_unfused_fwd(c, p, bt));
  } else if (p.fused_fe) {
    FrontArgs f = front_args(c, p, bt);
    f.dh = dxt;
    if (dxt == p.t_dx && first_unfused < 0) { f.dh = nullptr; f.dh_bf = reinterpret_cast<const bf16*>(p.t_dx); }
    f.dx0_part = p.dx0;                                  // partial dx0 between hidden passes (2D > 256)
    probe(PH_FE_MLP_BWD, 0, st); TRY(frontend_mlp_bwd(f, st)); probe(PH_FE_MLP_BWD, 1, st);
    join_side(st, ss);
    TRY((int)cudaGetLastError());
    return 0;
  }
  cast_rows_bf16(dxt, (int)T, d, d, p.dh_bf, d, p.real, st);
  TRY(lin_dx(st, p.dh_bf, d, T, p.pk.seq_w2, d, 2 * D, d, nullptr, 0, p.da1, 2 * D, p.a1));
  TRY(lin_dw(st, p.g1, 2 * D, 2 * D, p.dh_bf, d, d, T, c.g(o.seq_w2)));
  colsum_bf16(p.dh_bf, (int)T, d, d, c.g(o.seq_b2), st);
  TRY(lin_dx(st, p.da1, 2 * D, T, p.pk.seq_w1, 2 * D, d, 2 * D, p.dx0, d, p.dx0_bf, d, nullptr, p.real));
  TRY(lin_dw(st, p.x0, d, d, p.da1, 2 * D, 2 * D, T, c.g(o.seq_w1)));
  colsum_bf16(p.da1, (int)T, 2 * D, 2 * D, c.g(o.seq_b1), st);
  TRY(lin_dw(st, p.feat, p.FP, p.F, p.dx0_bf, d, d, T, c.g(o.tok_w)));
  colsum_f32(p.dx0, (int)T, d, d, c.g(o.tok_b), st);
  EmbedBwdArgs eb{};
  eb.items = bt.items; eb.actions = bt.actions; eb.dt = bt.dt; eb.n_events = bt.n_events;
  eb.B = p.B; eb.L = p.L; eb.Lp = p.Lp; eb.d = d; eb.d_item = dm.d_item; eb.d_act = dm.d_act; eb.d_time = dm.d_time;
  eb.nb = dm.n_time_buckets; eb.vocab = dm.vocab; eb.n_actions = dm.n_actions;
  eb.tok_w = c.w(o.tok_w); eb.dx0 = p.dx0;
  eb.g_item = c.g(o.item); eb.g_act = c.g(o.act); eb.g_time = c.g(o.time); eb.g_pos = c.g(o.pos);
  embed_bwd(eb, st);
  join_side(st, ss);
  TRY((int)cudaGetLastError());
  return 0;
}

bool use_fused(const Plan& p) {
  if (!g_knobs.fused) return false;
  return frontend_supported(p.d, p.K, p.D, p.F, p.IL) != 0 && p.dims.n_actions <= 32;
}

// The caller's batch with its per-sample ids replaced by range-checked copies in the workspace.
LongerBatch checked_batch(const Plan& p, const LongerBatch& bt, cudaStream_t st) {
  LongerBatch b = bt;
  check_sample_ids(bt.uid, bt.profile, bt.cand_item, p.B, p.dims.n_users, p.dims.n_profiles, p.dims.vocab, p.ids,
                   p.status, st);
  b.uid = p.ids;
  b.profile = p.ids + p.B;
  if (bt.cand_item) b.cand_item = p.ids + 2 * p.B;
  return b;
}

int check_call(const LongerDims* dims, size_t ws_bytes, Plan* out, void* ws) {
  g_err.clear();
  refresh_knobs();
  if (!dims) return fail(LONGER_EDIM, "null dims");
  int rc = validate(*dims);
  if (rc) return rc;
  *out = make_plan(*dims, ws);
  if (ws_bytes < out->bytes) return fail(LONGER_EDIM, "workspace too small");
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(LONGER_EDIM, "workspace must be 256-byte aligned");
  return 0;
}

// ------------------------------------------------------------------ serving (serving.py:84-167)
// Cache of U users (dims.batch), in one caller-owned buffer:
//   xkv  [U][v-1][2D] bf16  cross-layer [K | V] of the merged rows + the m-1 non-target globals
//   skv  [N][U][q-1][2D]    each self layer's [K | V] of the k seq queries + m-1 non-target globals
//   cls  [U][D] f32         CLS row of the last layer output (serving.py:141)
//   ud   [U][2d] f32        [uid_emb | profile_emb] (user_side_features)
//   npg  [U] i32            all-pad merged groups (the target's key mask, serving.py:137-139)
struct CacheLayout {
  size_t xkv, skv, cls, ud, npg, bytes;
  long long xrows, srows;
};

CacheLayout cache_layout(const Plan& p) {
  CacheLayout c{};
  const size_t U = p.B, D = p.D;
  c.xrows = p.v - 1;
  c.srows = p.q - 1;
  size_t off = 0;
  auto take = [&](size_t n) { off = (off + 255) & ~size_t(255); size_t r = off; off += n; return r; };
  c.xkv = take(U * c.xrows * 2 * D * 2);
  c.skv = take((size_t)p.N * U * c.srows * 2 * D * 2);
  c.cls = take(U * D * 4);
  c.ud = take(U * 2 * p.d * 4);
  c.npg = take(U * 4);
  c.bytes = (off + 255) & ~size_t(255);
  return c;
}

// Stage 1: the ordinary forward with a placeholder candidate, then keep the candidate-free rows.
// The visibility rule hides the target row from every other row (attention.py:49-87), so these
// rows are bit-identical to the ones the full forward of any candidate computes.
int cache_build(const Ctx& c, const Plan& p, const LongerBatch& user_batch, char* cache) {
  cudaStream_t st = c.st;
  const int D = p.D;
  LongerBatch bt = user_batch;
  TRY((int)cudaMemsetAsync(p.cand0, 0, sizeof(int32_t) * p.B, st));
  bt.cand_item = p.cand0;
  bt.label = nullptr;
  TRY(forward(c, p, bt, p.loss_per, nullptr, 0));
  const CacheLayout L = cache_layout(p);
  copy_rows_bf16(p.KV, (long long)p.v * 2 * D, 2 * D, 0, reinterpret_cast<bf16*>(cache + L.xkv), L.xrows * 2 * D,
                 (int)L.xrows, 2 * D, p.B, st);
  for (int i = 0; i < p.N; ++i) {
    bf16* dst = reinterpret_cast<bf16*>(cache + L.skv) + (size_t)i * p.B * L.srows * 2 * D;
    copy_rows_bf16(p.sb[i].qkv, (long long)p.q * 3 * D, 3 * D, D, dst, L.srows * 2 * D, (int)L.srows, 2 * D, p.B,
                   st);
  }
  CacheUserArgs u{};
  u.x_last = p.N ? p.sb[p.N - 1].out : p.cb.out;
  u.U = p.B; u.q = p.q; u.k = p.k; u.D = D; u.d = p.d;
  u.uid = user_batch.uid; u.profile = user_batch.profile; u.npg = p.npg;
  u.uid_tab = c.w(p.po.uid); u.prof_tab = c.w(p.po.prof);
  u.cls = reinterpret_cast<float*>(cache + L.cls);
  u.ud = reinterpret_cast<float*>(cache + L.ud);
  u.npg_out = reinterpret_cast<int32_t*>(cache + L.npg);
  cache_users(u, st);
  TRY((int)cudaGetLastError());
  return 0;
}

struct ScorePlan {
  Plan p;                      // dims (batch = users), packed weights, status
  int C;
  long long R;                 // users x candidates target rows
  bf16 *raw_bf, *gg, *qn, *qkv, *ctx, *x1n, *gf;
  float *x, *y, *m1, *r1, *x1, *m2, *r2;
  // per-item mode (vocab ≤ R / 4): the target row's path up to the cross attention depends on the
  // candidate item alone, so it runs once per vocabulary item and the candidates gather from it
  bool items;
  int V;
  bf16 *i_raw, *i_gg, *i_qn, *i_qkv;
  float *i_x, *i_m, *i_r;
  size_t bytes;
};

ScorePlan make_score_plan(const LongerDims& d, int C, void* ws) {
  ScorePlan s{};
  plan_dims(s.p, d, ws);
  Bump a{reinterpret_cast<char*>(ws)};
  s.p.status = a.take<int>(64);
  take_packed(s.p, a);
  s.C = C;
  s.R = (long long)d.batch * C;
  const long long R = s.R;
  const int D = s.p.D;
  s.raw_bf = a.take<bf16>(R * D); s.gg = a.take<bf16>(R * 2 * D);
  s.x = a.take<float>(R * D); s.y = a.take<float>(R * D);
  s.qn = a.take<bf16>(R * D); s.m1 = a.take<float>(R); s.r1 = a.take<float>(R);
  s.qkv = a.take<bf16>(R * 3 * D); s.ctx = a.take<bf16>(R * D);
  s.x1 = a.take<float>(R * D); s.x1n = a.take<bf16>(R * D); s.m2 = a.take<float>(R); s.r2 = a.take<float>(R);
  s.gf = a.take<bf16>(R * 4 * D);
  s.V = d.vocab;
  s.items = (long long)d.vocab * 4 <= R;
  if (s.items) {
    const long long V = d.vocab;
    s.i_raw = a.take<bf16>(V * D); s.i_gg = a.take<bf16>(V * 2 * D); s.i_qn = a.take<bf16>(V * D);
    s.i_qkv = a.take<bf16>(V * 3 * D); s.i_x = a.take<float>(V * D); s.i_m = a.take<float>(V);
    s.i_r = a.take<float>(V);
  }
  s.bytes = a.off + 256;
  return s;
}

// Y[rows, out] (bf16, row stride ldy) = X·W + bias
int lin_fwd_ld(cudaStream_t st, const bf16* X, int ldx, long long rows, const bf16* W, int in, int out,
               const float* bias, bf16* Y, int ldy) {
  GemmArgs g = G_(X, ldx, 0, W, out, 1, rows, out, in);
  g.flags = EPI_BIAS | EPI_OUT_BF16;
  g.bias = bias; g.C_bf16 = Y; g.ldc_bf = ldy;
  return gemm_launch(g, st);
}

// attention_block_cached (attention.py:215-236) for all R target rows: x → out.
// pre_done: [Q | K_own | V_own] of the rows are already in s.qkv (the per-item mode)
int serve_block(const Ctx& c, const ScorePlan& s, const BlockOff& bo, const float* x, float* out, bool cross,
                const bf16* kv, int nk, int ns, int goff, const int32_t* npg, const bf16* Wqkv, const float* bqkv,
                const bf16* Wo, const bf16* W1, const bf16* W2, bool pre_done = false) {
  const Plan& p = s.p;
  cudaStream_t st = c.st;
  const int D = p.D;
  const long long R = s.R;
  if (!pre_done) {
    layernorm_fwd(rows_plain(x, D, R), D, c.w(bo.ln1_g), c.w(bo.ln1_b), s.qn, s.m1, s.r1, st);
    if (cross) {   // cross weights are packed as W_q and [W_k | W_v]
      TRY(lin_fwd_ld(st, s.qn, D, R, p.pk.c_wq, D, D, c.w(bo.b_q), s.qkv, 3 * D));
      TRY(lin_fwd_ld(st, s.qn, D, R, p.pk.c_wkv, D, 2 * D, p.pk.c_bkv, s.qkv + D, 3 * D));
    } else {
      TRY(lin_fwd_ld(st, s.qn, D, R, Wqkv, D, 3 * D, bqkv, s.qkv, 3 * D));
    }
  }
  ServeAttnArgs a{};
  a.Q = s.qkv; a.ldq = 3 * D;
  a.Kown = s.qkv + D; a.Vown = s.qkv + 2 * D; a.ldown = 3 * D;
  a.K = kv; a.ldk = 2 * D; a.sk = (long long)nk * 2 * D;
  a.V = kv + D; a.ldv = 2 * D; a.sv = a.sk;
  a.U = p.B; a.C = s.C; a.nk = nk; a.ns = ns; a.goff = goff; a.D = D; a.heads = p.heads; a.npg = npg;
  a.ctx = s.ctx; a.ldc = D;
  TRY(serve_attn(a, st));
  TRY(lin_fwd(st, s.ctx, D, R, Wo, D, D, c.w(bo.b_o), 0, s.x1, nullptr, nullptr, x, D));
  layernorm_fwd(rows_plain(s.x1, D, R), D, c.w(bo.ln2_g), c.w(bo.ln2_b), s.x1n, s.m2, s.r2, st);
  TRY(lin_fwd(st, s.x1n, D, R, W1, D, 4 * D, c.w(bo.b1), EPI_GELU, nullptr, s.gf, nullptr));
  TRY(lin_fwd(st, s.gf, 4 * D, R, W2, 4 * D, D, c.w(bo.b2), 0, out, nullptr, nullptr, s.x1, D));
  return 0;
}

// Stage 2: candidates → target global rows → cross + N self blocks against the cache → head.
int cache_score(const Ctx& c, const ScorePlan& s, const char* cache, const int32_t* cand, float* probs) {
  const Plan& p = s.p;
  cudaStream_t st = c.st;
  const ParamOff& o = p.po;
  const LongerDims& dm = p.dims;
  const int D = p.D;
  const long long R = s.R;
  const CacheLayout L = cache_layout(p);
  TRY(pack_weights(p, c.P, p.ws, st));
  TargetArgs t{};
  t.d = p.d; t.D = D; t.d_item = dm.d_item; t.d_act = dm.d_act; t.d_time = dm.d_time;
  t.vocab = dm.vocab; t.item_tab = c.w(o.item); t.time_tab = c.w(o.time); t.tok_w = c.w(o.tok_w);
  t.tok_b = c.w(o.tok_b); t.lift_w = c.w(o.lift_w); t.lift_b = c.w(o.lift_b);
  t.status = p.status;
  if (s.items) {
    // target_global_token → global MLP → cross LN1 → [Q | K_own | V_own] once per vocabulary item
    // (the row depends on the candidate item alone), then one gather per candidate
    const long long V = s.V;
    t.cand = nullptr; t.R = V; t.raw_bf = s.i_raw;
    target_rows(t, st);
    TRY(lin_fwd(st, s.i_raw, D, V, p.pk.glob_w1, D, 2 * D, c.w(o.glob_b1), EPI_GELU, nullptr, s.i_gg, nullptr));
    TRY(lin_fwd(st, s.i_gg, 2 * D, V, p.pk.glob_w2, 2 * D, D, c.w(o.glob_b2), 0, s.i_x, nullptr, nullptr));
    layernorm_fwd(rows_plain(s.i_x, D, V), D, c.w(o.cross.ln1_g), c.w(o.cross.ln1_b), s.i_qn, s.i_m, s.i_r, st);
    TRY(lin_fwd_ld(st, s.i_qn, D, V, p.pk.c_wq, D, D, c.w(o.cross.b_q), s.i_qkv, 3 * D));
    TRY(lin_fwd_ld(st, s.i_qn, D, V, p.pk.c_wkv, D, 2 * D, p.pk.c_bkv, s.i_qkv + D, 3 * D));
    gather_item_rows(cand, R, dm.vocab, s.i_x, s.i_qkv, D, s.x, s.qkv, p.status, st);
  } else {
    t.cand = cand; t.R = R; t.raw_bf = s.raw_bf;
    target_rows(t, st);
    TRY(lin_fwd(st, s.raw_bf, D, R, p.pk.glob_w1, D, 2 * D, c.w(o.glob_b1), EPI_GELU, nullptr, s.gg, nullptr));
    TRY(lin_fwd(st, s.gg, 2 * D, R, p.pk.glob_w2, 2 * D, D, c.w(o.glob_b2), 0, s.x, nullptr, nullptr));
  }
  const int32_t* npg = reinterpret_cast<const int32_t*>(cache + L.npg);
  float* x = s.x;
  float* y = s.y;
  TRY(serve_block(c, s, o.cross, x, y, true, reinterpret_cast<const bf16*>(cache + L.xkv), (int)L.xrows, p.G, 0, npg,
                  nullptr, nullptr, p.pk.c_wo, p.pk.c_w1, p.pk.c_w2, s.items));
  std::swap(x, y);
  for (int i = 0; i < p.N; ++i) {
    const bf16* kv = reinterpret_cast<const bf16*>(cache + L.skv) + (size_t)i * p.B * L.srows * 2 * D;
    // the target sees every non-pad sequence query: key j is pad iff (G-k)+j < npg, never for the bank
    const int goff = p.qs == QS_LEARNABLE ? p.G : p.G - p.k;
    TRY(serve_block(c, s, o.self_[i], x, y, false, kv, (int)L.srows, p.k, goff, npg, p.pk.s_wqkv[i],
                    p.pk.s_bqkv[i], p.pk.s_wo[i], p.pk.s_w1[i], p.pk.s_w2[i]));
    std::swap(x, y);
  }
  ServeHeadArgs h{};
  h.x = x; h.R = R; h.C = s.C; h.D = D; h.d = p.d; h.hh = p.hh;
  h.cls = reinterpret_cast<const float*>(cache + L.cls);
  h.ud = reinterpret_cast<const float*>(cache + L.ud);
  h.w1 = c.w(o.head_w1); h.b1 = c.w(o.head_b1); h.w2 = c.w(o.head_w2); h.b2 = c.w(o.head_b2);
  h.probs = probs;
  serve_head(h, st);
  TRY((int)cudaGetLastError());
  return 0;
}

}  // namespace
}  // namespace longer

using namespace longer;

extern "C" int longer_param_count(const LongerDims* dims, int64_t* count) {
  if (!dims || !count) return fail(LONGER_EDIM, "null argument");
  int rc = validate(*dims);
  if (rc) return rc;
  *count = param_offsets(*dims).total;
  return 0;
}

extern "C" int longer_workspace_bytes(const LongerDims* dims, size_t* bytes) {
  if (!dims || !bytes) return fail(LONGER_EDIM, "null argument");
  int rc = validate(*dims);
  if (rc) return rc;
  *bytes = make_plan(*dims, nullptr).bytes;
  return 0;
}

// training / inference entry points run the last self block's tail on the two head rows
// (LONGER_HEAD_ROWS=0: all rows); the serving cache build keeps every row (it caches them)
static bool compact_head_ok(const Plan& p) {
  return p.N >= 1 && p.m >= 3 && g_knobs.head_rows;
}
// absorbed cross-layer K/V projections: one head (per-head absorption would widen every head to D)
// on the tensor-core attention; the serving cache build keeps explicit K/V rows (it caches them)
static bool absorb_ok(const Plan& p) {
  const bool tc = (p.q <= 128 && (p.D == 32 || p.D == 64 || p.D == 128)) || (p.q <= 64 && p.D == 256);
  return g_knobs.absorb_kv && g_knobs.attn_tc && p.heads == 1 && tc;
}

extern "C" int longer_forward(const LongerDims* dims, const float* params, const LongerBatch* batch, void* ws,
                              size_t ws_bytes, float* probs, void* stream) {
  Plan p;          // per call: no state survives between calls (re-entrant)
  int rc = check_call(dims, ws_bytes, &p, ws);
  if (rc) return rc;
  p.fused_fe = use_fused(p);
  p.compact_head = compact_head_ok(p);
  p.absorb = absorb_ok(p);
  Ctx c{p, params, nullptr, (cudaStream_t)stream};
  return forward(c, p, checked_batch(p, *batch, c.st), probs, nullptr, 0);
}

extern "C" int longer_forward_trace(const LongerDims* dims, const float* params, const LongerBatch* batch,
                                    void* ws, size_t ws_bytes, float* probs, LongerTrace* trace, void* stream) {
  Plan p;
  int rc = check_call(dims, ws_bytes, &p, ws);
  if (rc) return rc;
  if (!batch || !probs || !trace) return fail(LONGER_EDIM, "null argument");
  p.fused_fe = use_fused(p);
  p.compact_head = false;                // every row of every layer is kept for the trace
  p.absorb = absorb_ok(p);
  Ctx c{p, params, nullptr, (cudaStream_t)stream};
  rc = forward(c, p, checked_batch(p, *batch, c.st), probs, nullptr, 0);
  if (rc) return rc;
  LongerTrace t{};
  t.h = p.IL ? p.h : p.merged;
  t.merged = p.merged;
  t.query_groups = (p.qs == QS_UNIFORM || p.qs == QS_RECENT_UNIFORM) ? p.qg : nullptr;
  t.n_layers = 1 + p.N;
  t.layers[0] = p.cb.out;
  for (int i = 0; i < p.N; ++i) t.layers[1 + i] = p.sb[i].out;
  t.head_input = p.hin;
  t.Lp = p.Lp; t.G = p.G; t.q = p.q; t.head_width = p.HIN;
  *trace = t;
  return 0;
}

extern "C" int longer_forward_backward(const LongerDims* dims, const float* params, const LongerBatch* batch,
                                       void* ws, size_t ws_bytes, float* probs, float* loss, float* grads,
                                       void* stream) {
  Plan p;
  int rc = check_call(dims, ws_bytes, &p, ws);
  p.fused_fe = use_fused(p);
  if (rc) return rc;
  p.compact_head = compact_head_ok(p);
  p.absorb = absorb_ok(p);
  Ctx c{p, params, grads, (cudaStream_t)stream};
  // the per-sample id check on the side stream: its first readers (the global tokens) run there, the
  // main stream reaches the ids only after waiting for them (head), and the call ends joined
  const cudaStream_t ss = side_stream(c.st);
  fork_side(c.st, ss);
  const LongerBatch bt = checked_batch(p, *batch, ss);
  rc = forward(c, p, bt, probs, loss, 1);
  if (rc) return rc;
  return backward(c, p, bt, probs);
}

extern "C" int longer_backward(const LongerDims* dims, const float* params, const LongerBatch* batch, void* ws,
                               size_t ws_bytes, const float* probs, const float* dprobs, float* grads, void* stream) {
  Plan p;
  int rc = check_call(dims, ws_bytes, &p, ws);
  if (rc) return rc;
  if (!batch || !probs || !dprobs || !grads) return fail(LONGER_EDIM, "null argument");
  p.fused_fe = use_fused(p);
  p.compact_head = compact_head_ok(p);
  p.absorb = absorb_ok(p);
  Ctx c{p, params, grads, (cudaStream_t)stream};
  dz_from_dprobs(probs, dprobs, p.B, p.dz, c.st);     // dL/dz = dL/dp · p(1 − p)
  return backward(c, p, checked_batch(p, *batch, c.st), const_cast<float*>(probs));
}

extern "C" int longer_adam_step(float* params, const float* grads, float* m, float* v, int64_t count, float lr,
                                int32_t t, void* stream) {
  if (t < 1) return fail(LONGER_ECONFIG, "Adam step counter must be >= 1");
  adam_step(params, grads, m, v, count, lr, t, (cudaStream_t)stream);
  int e = (int)cudaGetLastError();
  return e ? fail(LONGER_ECUDA, cudaGetErrorString((cudaError_t)e)) : 0;
}

extern "C" int longer_read_status(void* ws, int32_t* flags, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int e = (int)cudaMemcpyAsync(flags, ws, 4, cudaMemcpyDeviceToHost, st);
  if (!e) e = (int)cudaStreamSynchronize(st);
  if (!e) e = (int)cudaMemsetAsync(ws, 0, 4, st);
  return e ? fail(LONGER_ECUDA, cudaGetErrorString((cudaError_t)e)) : 0;
}

extern "C" const char* longer_last_error(void) { return g_err.c_str(); }

extern "C" int longer_cache_bytes(const LongerDims* dims, size_t* bytes) {
  if (!dims || !bytes) return fail(LONGER_EDIM, "null argument");
  int rc = validate(*dims);
  if (rc) return rc;
  Plan p{};
  plan_dims(p, *dims, nullptr);
  *bytes = cache_layout(p).bytes;
  return 0;
}

extern "C" int longer_cache_build(const LongerDims* dims, const float* params, const LongerBatch* batch, void* ws,
                                  size_t ws_bytes, void* cache, size_t cache_bytes, void* stream) {
  Plan p;
  int rc = check_call(dims, ws_bytes, &p, ws);
  if (rc) return rc;
  if (!batch || !cache) return fail(LONGER_EDIM, "null batch or cache");
  if (cache_bytes < cache_layout(p).bytes) return fail(LONGER_EDIM, "cache buffer too small");
  p.fused_fe = use_fused(p);
  Ctx c{p, params, nullptr, (cudaStream_t)stream};
  return cache_build(c, p, checked_batch(p, *batch, c.st), reinterpret_cast<char*>(cache));
}

extern "C" int longer_score_workspace_bytes(const LongerDims* dims, int32_t candidates_per_user, size_t* bytes) {
  if (!dims || !bytes) return fail(LONGER_EDIM, "null argument");
  int rc = validate(*dims);
  if (rc) return rc;
  if (candidates_per_user < 1) return fail(LONGER_EDIM, "candidates_per_user must be >= 1");
  *bytes = make_score_plan(*dims, candidates_per_user, nullptr).bytes;
  return 0;
}

extern "C" int longer_cache_score(const LongerDims* dims, const float* params, const void* cache, size_t cache_bytes,
                                  const int32_t* cand_items, int32_t candidates_per_user, void* ws, size_t ws_bytes,
                                  float* probs, void* stream) {
  g_err.clear();
  if (!dims || !cache || !cand_items || !probs) return fail(LONGER_EDIM, "null argument");
  int rc = validate(*dims);
  if (rc) return rc;
  if (candidates_per_user < 1) return fail(LONGER_EDIM, "candidates_per_user must be >= 1");
  refresh_knobs();
  // the serving chain has no fused front-end kernels; its GEMM boundaries gain from early launch
  // (c4: 73.4 M candidates/s without fences, 68.8 M with the training default)
  if (!std::getenv("LONGER_PDL_FENCE")) g_knobs.pdl_fence = 0;
  ScorePlan s = make_score_plan(*dims, candidates_per_user, ws);
  if (ws_bytes < s.bytes) return fail(LONGER_EDIM, "workspace too small");
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(LONGER_EDIM, "workspace must be 256-byte aligned");
  if (cache_bytes != cache_layout(s.p).bytes)
    return fail(LONGER_ESTALE, "cache was built for different dimensions (rebuild it)");
  Ctx c{s.p, params, nullptr, (cudaStream_t)stream};
  return cache_score(c, s, reinterpret_cast<const char*>(cache), cand_items, probs);
}

extern "C" int longer_grad_early_begin(const LongerDims* dims, int64_t* begin) {
  if (!dims || !begin) return fail(LONGER_EDIM, "null argument");
  int rc = validate(*dims);
  if (rc) return rc;
  *begin = param_offsets(*dims).cross.w_q;
  return 0;
}

extern "C" int longer_set_grad_event(void* ev) {
  g_grad_event = (cudaEvent_t)ev;
  return 0;
}

extern "C" int longer_set_probe(int32_t phase, void* ev_begin, void* ev_end) {
  if (phase < 0 || phase >= PH_N) return fail(LONGER_EDIM, "unknown probe phase");
  g_probe[phase][0] = (cudaEvent_t)ev_begin;
  g_probe[phase][1] = (cudaEvent_t)ev_end;
  return 0;
}
