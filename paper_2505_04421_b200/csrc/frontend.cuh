// frontend.cuh — fused token front-end (ids → merged rows) for sm_100a, forward and backward.
//
// One persistent CTA walks 128-token tiles.  Every dense stage is a tcgen05 MMA (M = 128 tokens)
// whose A operand the worker warps write into shared memory in the canonical no-swizzle layout,
// with the weights resident in shared memory (packed once per step) and the accumulator in TMEM.
// Nothing between the ids and the merged row touches HBM; the backward recomputes each tile
// and keeps the front-end weight gradients in TMEM for the whole kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace longer {

struct FrontArgs {
  // batch
  const int32_t *items, *actions, *dt, *n_events;
  int B, L, Lp, K, d, d_item, d_act, d_time, nb, vocab, n_actions, inner_layers;
  int item_smem = 1;           // fe_mlp_bwd: stage the item-table gradient in shared memory when it fits
  // fe_mlp_bwd hidden passes (set by frontend_mlp_bwd): this launch covers hidden units
  // [mlp_h0, mlp_h0 + mlp_hn) of the 2D; mlp_last: it finishes dx0 (the featuriser / table part);
  // dx0_part: [T, d] fp32 partial dx0 carried between passes (read when mlp_h0 > 0, written when
  // not the last pass)
  int mlp_h0 = 0, mlp_hn = 0, mlp_last = 1;
  // mlp_split: fe_mlp_bwd's CTAs take equal ranges of the column-block-major tile order instead of
  // one column block each (long sequences: more column blocks than SMs would leave idle)
  int mlp_split = 0;
  // fe_fwd: the cross-LN1 gain / bias read from global memory (L1) instead of shared memory, which
  // lets c5's D = 256 fit a fourth tile slot
  int kn_global = 0;
  float* dx0_part = nullptr;
  long long T;                 // B * Lp tokens
  // fp32 master parameters (biases, tables)
  const float *item_tab, *act_tab, *time_tab, *pos_tab, *tok_w, *tok_b, *seq_b1, *seq_b2;
  const float* inner_bias[8][6];   // per layer: b_q, b_k, b_v, b_o, b1, b2
  const float* inner_ln[8][4];     // per layer: ln1_g, ln1_b, ln2_g, ln2_b
  // packed bf16 weight blob (see pack_frontend_weights)
  const bf16* wblob;
  // the embedding tables projected through tok_proj (fp32): rows [0, vocab) item_table·W_tp[item
  // cols], then n_actions rows action_table·W_tp[action cols], then nb rows
  // time_table·W_tp[time cols] + b_tp — so x0 = P[item] + P[action] + P[bucket] + abs_pos
  const float* proj;
  // forward outputs
  float* merged;               // [T, d]  (== [B*G, D])
  float* h_out;                // [T, d]  token-MLP output (InnerTrans input), saved for backward (or null)
  int* status;
  int32_t* npg;                // [B] all-pad merged groups per sample
  float *real_out, *keep_out;  // [T] token is real / token's group is not all-pad (or null)
  // optional fused epilogue: the cross block's LN1 of every merged row (a group of K tokens),
  // written as the bf16 K/V-projection operand kn[b*v + g] with its mean / rstd
  const float *kn_g, *kn_b;
  bf16* kn;
  float *kn_mean, *kn_rstd;
  int v;                       // rows per sample in kn (G + m)
  // backward
  const float* dh;             // [T, d] gradient w.r.t. the token-MLP output (MLP backward input)
  const bf16* dh_bf = nullptr; // or the same in bf16 (the InnerTrans backward's output): read instead
                               // of dh — the MLP backward takes it as a bf16 MMA operand anyway
  float *g_tok_w, *g_tok_b, *g_seq_w1, *g_seq_b1, *g_seq_w2, *g_seq_b2;
  float *g_item, *g_act, *g_time, *g_pos;
  // InnerTrans backward (layer 0): h saved by the forward, dmerged in, dh out
  const float* h_in;           // [T, d]
  const float* dmerged;        // [T, d]
  float* dh_out;               // [T, d]
  bf16* dh_out_bf = nullptr;   // [T, d] bf16 instead of dh_out (when the fused MLP backward reads it)
  float* g_inner[16];          // grads of w_q,b_q,w_k,b_k,w_v,b_v,w_o,b_o,w1,b1,w2,b2,ln1_g,ln1_b,ln2_g,ln2_b
};

int frontend_blob_bytes(int d, int D, int inner_layers);
// inner_w[l] = param offsets of {w_q, w_k, w_v, w_o} of InnerTrans layer l (w1, w2 follow the
// reference order after b_o).
// P (see FrontArgs::proj) from the fp32 master tables: (vocab + n_actions + nb) x d floats,
// computed by the same launch as the weight blob
struct ProjArgs {
  const float *item_tab, *act_tab, *time_tab, *tok_w, *tok_b;
  int vocab, n_actions, nb, d_item, d_act, d_time, d;
  float* proj;
};
void pack_frontend_weights(const float* params, long long tok_w, long long seq_w1, long long seq_w2,
                           const long long (*inner_w)[4], int d, int D, int F, int inner_layers, bf16* blob,
                           const ProjArgs& pj, cudaStream_t st);

int frontend_supported(int d, int K, int D, int F, int inner_layers);
// the fused token-MLP backward takes 2D ≤ 256 in one pass, or 2D a multiple of 256 in passes of
// 256 hidden units (TMEM / shared-memory budget per pass); FrontArgs::dx0_part must be set then
int frontend_mlp_bwd_supported(int d, int K, int D);
int frontend_fwd(const FrontArgs& a, cudaStream_t st);
// token-MLP + featuriser backward: dh → all front-end MLP/featuriser/table/pos gradients
int frontend_mlp_bwd(const FrontArgs& a, cudaStream_t st);
// InnerTrans (one layer) backward: recompute the layer from h, dmerged → dh + layer gradients
int frontend_inner_bwd(const FrontArgs& a, cudaStream_t st);

}  // namespace longer
