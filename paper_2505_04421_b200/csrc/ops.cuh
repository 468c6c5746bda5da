// ops.cuh — launchers of the non-GEMM kernels (embedding, norms, attention, head, globals).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace longer {

// ---------------------------------------------------------------- front-end (tokens)
struct EmbedArgs {
  const int32_t *items, *actions, *dt, *n_events;
  int B, L, Lp, d, d_item, d_act, d_time, FP, nb, vocab, n_actions;
  const float *item_tab, *act_tab, *time_tab, *pos_tab, *tok_w, *tok_b;   // fp32 master
  bf16* feat;        // [T, FP]  concat(item, act, time) embedding, zero-padded to FP
  bf16* x0;          // [T, d]   feat·W_tp + b_tp + abs_pos[recency]   (0 for pad tokens)
  float* real;       // [T]      1 real / 0 pad
  float* keep;       // [T]      1 unless the token's merged group is all padding
  int K;
  int* status;       // bit0 id out of range, bit1 negative delta
  int32_t* npg;      // [B] all-pad merged groups per sample ((Lp - n) // K)
};
void embed_fwd(const EmbedArgs& a, cudaStream_t st);

struct EmbedBwdArgs {
  const int32_t *items, *actions, *dt, *n_events;
  int B, L, Lp, d, d_item, d_act, d_time, nb, vocab, n_actions;
  const float* tok_w;        // [F, d]
  const float* dx0;          // [T, d] fp32 (already masked to real tokens)
  float *g_item, *g_act, *g_time, *g_pos;
};
void embed_bwd(const EmbedBwdArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- row layer norm
// Rows are addressed through a two-source remap so LN can read R = [merged; globals] or
// O = [merged[G-k:]; globals] without materialising them:
//   for batch b, output row j (< na + nb):  j < na → A[(b*a_rows + a_off + j) * lda]
//                                            else  → Bsrc[(b*nb + j - na) * ldb]
struct RowMap {
  const float* A; int lda; int a_rows; int a_off; int na;
  const float* Bsrc; int ldb; int nb;
  int batch;
  // layernorm_fwd output placement: row b*(na+nb)+j goes to b*o_per + o_off + j (o_per = 0: same row)
  int o_per, o_off;
  __host__ __device__ int rows() const { return batch * (na + nb); }
  __host__ __device__ int out_row(int row) const {
    return o_per ? (row / (na + nb)) * o_per + o_off + row % (na + nb) : row;
  }
};
// y = LN(x)·g + b  → bf16 [rows, W]; mean/rstd saved; xcopy (optional): the input rows, fp32 [rows, W]
void layernorm_fwd(const RowMap& x, int W, const float* g, const float* b, bf16* y, float* mean, float* rstd,
                   cudaStream_t st, float* xcopy = nullptr);
// out(remap-writable) (+)= LN_bw(dy); dgain/dbias accumulated (atomic) into grads.
struct RowMapW {
  float* A; int lda; int a_rows; int a_off; int na;
  float* Bsrc; int ldb; int nb;
  int batch;
};
// Optional extras of the LN backward (plain row indexing, row stride W):
//   addend     out += addend[row]           (the residual branch's gradient)
//   out_bf     bf16 copy of out              (the next GEMM's operand)
//   colsum_out += column sums of out         (the bias gradient of the linear layer feeding out)
struct LnBwdExtra {
  const float* addend = nullptr;
  bf16* out_bf = nullptr;
  float* colsum_out = nullptr;
};
void layernorm_bwd(const RowMap& x, int W, const float* g, const float* mean, const float* rstd,
                   const float* dy, int ldy, const RowMapW& out, int accumulate, const float* rowmask,
                   float* dgain, float* dbias, cudaStream_t st, LnBwdExtra ex = LnBwdExtra());

// the same with a bf16 dy and no extras (W ≤ 256)
void layernorm_bwd(const RowMap& x, int W, const float* g, const float* mean, const float* rstd,
                   const bf16* dy, int ldy, const RowMapW& out, float* dgain, float* dbias, cudaStream_t st);

// column sums of a [rows, W] matrix (fp32 or bf16), atomically added to out[W]
void colsum_f32(const float* x, int rows, int W, int ld, float* out, cudaStream_t st);
void colsum_bf16(const bf16* x, int rows, int W, int ld, float* out, cudaStream_t st);

// elementwise helpers
void cast_rows_bf16(const float* x, int rows, int W, int ldx, bf16* y, int ldy, const float* rowmask,
                    cudaStream_t st);
void mul_rows_inplace(float* x, int rows, int W, const float* rowmask, cudaStream_t st);
void gather_rows_f32(const float* src, int batch, int src_rows, int src_off, int n, float* dst_base,
                     int dst_rows, int dst_off, int W, cudaStream_t st);
void add_rows_f32(const float* src, int batch, int src_rows, int src_off, int n, float* dst_base,
                  int dst_rows, int dst_off, int W, cudaStream_t st);

// ---------------------------------------------------------------- attention
// grouped (InnerTrans) attention: groups of K consecutive rows, no mask, scale 1/sqrt(w)
void group_attn_fwd(const float* qkv, int T, int K, int w, bf16* ctx, float* probs, cudaStream_t st);
void group_attn_bwd(const float* qkv, const float* probs, const float* dctx, int T, int K, int w, bf16* dqkv,
                    cudaStream_t st);

// hybrid (cross/self) attention per sample with the VisRule mask.
struct AttnArgs {
  const bf16* Q; int ldq; long long sq;     // per-sample stride (elements)
  const bf16* Kp; int ldk; long long sk;
  const bf16* V; int ldv; long long sv;
  int nq, nk, D, heads;
  int k, G, ns, goff;                        // VisRule parameters
  const int32_t* qg;                         // [B, k] query groups (nullptr: "recent")
  int learn, self_keys;                      // "learnable" bank; self layer (keys = query rows)
  const int32_t* npg;                        // [B] pad groups
  int B;
  bf16* ctx; int ldc; long long sc;          // fwd out (GEMM operand)
  float* ctx32;                              // fwd out fp32 copy, same ld/stride (bwd D_i)
  float* lse;                                // [B, heads, nq] (−inf for fully masked rows)
  // backward
  const float* dctx; int lddc; long long sdc;
  const bf16* ctx_in;                        // forward context (for D_i)
  bf16* dQ; int lddq; long long sdq;
  bf16* dK; int lddk; long long sdk;
  bf16* dV; int lddv; long long sdv;
  int sum_kv;                                // K and V are the same rows (absorbed projections):
                                             // dK + dV go to dK (tensor-core path only)
};
void attn_fwd(const AttnArgs& a, cudaStream_t st);
void attn_bwd(const AttnArgs& a, cudaStream_t st);
// tcgen05 versions for the cross layer (attn_tc.cu): q ≤ 128 query rows, head width 32/64/128
int attn_tc_supported(const AttnArgs& a);
int attn_tc_fwd(const AttnArgs& a, cudaStream_t st);
int attn_tc_bwd(const AttnArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- query selection (model.py:58-123)
// qg[b, 0..k) = the merged groups of sample b's sequence queries for strategy
// 1 = uniform, 3 = recent_uniform (0 = recent and 2 = learnable need no table)
void select_queries(const int32_t* npg, int B, int G, int k, int strategy, int32_t* qg, cudaStream_t st);
// O[b, i] = merged[b, qg[b, i]] (or bank[i] when bank != nullptr), rows of width W, i < k
void gather_query_rows(const float* merged, const int32_t* qg, const float* bank, int B, int G, int k, int W,
                       float* O, int q, cudaStream_t st);
// dmerged[b, qg[b, i]] += dO[b, i]  (or g_bank[i] += Σ_b dO[b, i] when g_bank != nullptr)
void scatter_query_rows(const float* dO, int q, const int32_t* qg, int B, int G, int k, int W, float* dmerged,
                        float* g_bank, cudaStream_t st);

// ---------------------------------------------------------------- globals + head
struct GlobalsArgs {
  const int32_t *uid, *cand_item;
  int B, m, d, D, d_item, d_act, d_time;
  const float *uid_tab, *item_tab, *time_tab, *cls, *tok_w, *tok_b, *lift_w, *lift_b;
  float* raw;      // [B*m, D] fp32
  bf16* raw_bf;    // [B*m, D]
  float* td;       // [B, d]   target featurizer output (pre-lift)
  // backward
  const float* draw;   // [B*m, D]
  float *g_uid, *g_item, *g_time, *g_cls, *g_tok_w, *g_tok_b, *g_lift_w, *g_lift_b;
};
void globals_raw_fwd(const GlobalsArgs& a, cudaStream_t st);

// _checked_ids for the per-sample ids (pkg/src/longrec/inputs.py:406-411): out[0:B) uid,
// out[B:2B) profile, out[2B:3B) candidate item — each copied, or 0 with status bit 0 set when out
// of range, so no kernel ever reads outside a table and the call reports EmbeddingLookupError.
void check_sample_ids(const int32_t* uid, const int32_t* profile, const int32_t* cand, int B, int n_users,
                      int n_profiles, int vocab, int32_t* out, int* status, cudaStream_t st);
void globals_raw_bwd(const GlobalsArgs& a, cudaStream_t st);

struct HeadArgs {
  const float* x;      // [B*q, D] final layer output
  int B, q, k, m, D, d, hh;
  const int32_t *uid, *profile;
  const float *label, *uid_tab, *prof_tab, *w1, *b1, *w2, *b2;
  float* hin;          // [B, 4D+2d]
  float* z1;           // [B, hh]
  float* probs;        // [B]
  float* loss_per;     // [B]
  float* dz;           // [B]
  float* loss;         // [1] batch mean
  // backward
  float* dx;           // [B*q, D]  (zeroed by caller) ← head grads into rows k+m-1 and k+1
  bf16* dx_bf;         // optional bf16 copy of dx (zeroed by caller), same two rows written
  float *g_w1, *g_b1, *g_w2, *g_b2, *g_uid, *g_prof;
  float* dz1;          // [B, hh] scratch
};
void head_fwd(const HeadArgs& a, int with_loss, cudaStream_t st);
void loss_mean(const float* loss_per, int B, float* loss, cudaStream_t st);   // batch-mean BCE
// dz[b] = dprobs[b] · p(1 − p): the head's logit gradient for an arbitrary upstream dL/dp
void dz_from_dprobs(const float* probs, const float* dprobs, int B, float* dz, cudaStream_t st);
void head_bwd(const HeadArgs& a, cudaStream_t st);
// the head's weight / table gradients from head_bwd's dz1 (feeds only the gradient buffer)
void head_wgrad(const HeadArgs& a, cudaStream_t st);
// the two head rows of each sample (r0 = k+1, r1 = k+m−1) between a full [B·q, W] buffer and a
// compact [2B, W] one (the scatter writes every row of `full`: zero outside the head rows)
void head_rows_gather_f32(const float* full, float* compact, int B, int q, int r0, int r1, int W, cudaStream_t st);
void head_rows_gather_bf16(const bf16* full, bf16* compact, int B, int q, int r0, int r1, int W, cudaStream_t st);
void head_rows_scatter_f32(const float* compact, float* full, int B, int q, int r0, int r1, int W, cudaStream_t st);
// the two gathers (bf16 context rows + fp32 residual rows) / the two scatters in one launch each
void head_rows_gather_pair(const bf16* full_b, bf16* compact_b, const float* full_f, float* compact_f, int B, int q,
                           int r0, int r1, int W, cudaStream_t st);
void head_rows_scatter_pair(const float* c0, float* f0, const float* c1, float* f1, int B, int q, int r0, int r1,
                            int W, cudaStream_t st);

// ---------------------------------------------------------------- weights
// Packs fp32 master parameters into the bf16 / fp32 operand layouts the kernels use.
struct CopySpec {
  int src_off;    // element offset into params
  int dst_off;    // element offset into the destination buffer
  int rows, cols, src_ld, dst_ld;
  int to_bf16;    // 1: bf16 destination, 0: fp32
};
constexpr int kMaxPackSpecs = 256;
struct PackList {
  int n;
  CopySpec s[kMaxPackSpecs];
};
void pack_params(const float* params, const PackList& specs, void* dst_base, cudaStream_t st);

void adam_step(float* p, const float* g, float* m, float* v, long long n, float lr, int t, cudaStream_t st);

}  // namespace longer
