// frontend.cuh — fused token front-end (ids → merged rows) for sm_100a.
//
// One persistent CTA walks 128-token tiles.  Every dense stage is a tcgen05 MMA (M = 128 tokens)
// whose A operand the worker warps write into shared memory in the canonical no-swizzle K-major
// layout, with the weights resident in shared memory (packed once per step in the same layout)
// and the accumulator in TMEM.  Nothing between the ids and the merged row touches HBM.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace longer {

struct FrontArgs {
  // batch
  const int32_t *items, *actions, *dt, *n_events;
  int B, L, Lp, K, d, d_item, d_act, d_time, nb, vocab, n_actions, inner_layers;
  long long T;                 // B * Lp tokens
  // fp32 master parameters (biases, tables)
  const float *item_tab, *act_tab, *time_tab, *pos_tab, *tok_b, *seq_b1, *seq_b2;
  const float* inner_bias[8][8];   // per layer: b_q, b_k, b_v, b_o, b1, b2, ln1 (g,b) .. see frontend.cu
  const float* inner_ln[8][4];     // ln1_g, ln1_b, ln2_g, ln2_b
  // packed bf16 weight blob (canonical K-major layout, see pack_frontend_weights)
  const bf16* wblob;
  int wblob_bytes;
  // outputs
  float* merged;               // [T, d]  (== [B*G, D])
  int* status;
  int32_t* npg;                // [B] all-pad merged groups per sample
  // backward
  const float* dmerged;        // [T, d]
  float* gW;                   // fp32 grads, same flat layout as params (front-end slots only)
  long long g_tok_w, g_tok_b, g_seq_w1, g_seq_b1, g_seq_w2, g_seq_b2, g_item, g_act, g_time, g_pos;
  long long g_inner[8][16];    // per inner layer: offsets of w_q.. ln2_b in the reference order
};

// Packs the front-end weights into the canonical blob.  Returns the blob size in bytes
// (call with dst = nullptr to size it).
int frontend_blob_bytes(int d, int D, int F, int inner_layers);
void pack_frontend_weights(const float* params, long long tok_w, long long seq_w1, long long seq_w2,
                           const long long (*inner_w)[4], int d, int D, int F, int inner_layers, bf16* blob,
                           cudaStream_t st);

// Returns 1 when the fused path supports the configuration.
int frontend_supported(int d, int K, int D, int F, int inner_layers);
int frontend_fwd(const FrontArgs& a, cudaStream_t st);

}  // namespace longer
