// serve.cuh — KV-cache serving kernels (serve.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace longer {

// copy `rows` x `cols` bf16 sub-blocks of `batch` matrices: dst[u][r][c] = src[u*s_stride + r*s_ld + s_col + c]
void copy_rows_bf16(const bf16* src, long long s_stride, int s_ld, int s_col, bf16* dst, long long d_stride, int rows,
                    int cols, int batch, cudaStream_t st);

struct CacheUserArgs {
  const float* x_last;        // [U*q, D] last-layer output of the cache-build forward
  int U, q, k, D, d;
  const int32_t *uid, *profile, *npg;
  const float *uid_tab, *prof_tab;
  float* cls;                 // [U, D]
  float* ud;                  // [U, 2d]
  int32_t* npg_out;           // [U]
};
void cache_users(const CacheUserArgs& a, cudaStream_t st);

struct TargetArgs {
  const int32_t* cand;        // [R] candidate items (nullptr: row r is item r)
  long long R;
  int d, D, d_item, d_act, d_time, vocab;
  const float *item_tab, *time_tab, *tok_w, *tok_b, *lift_w, *lift_b;
  bf16* raw_bf;               // [R, D]
  int* status;
};
void target_rows(const TargetArgs& a, cudaStream_t st);

// per-candidate rows from per-item tables (the candidate-only part of the target row's path):
// x[r] = item_x[cand[r]] (fp32, D), qkv[r] = item_qkv[cand[r]] (bf16, 3D); out-of-range ids flag
// status bit 0 and read item 0
void gather_item_rows(const int32_t* cand, long long R, int vocab, const float* item_x, const bf16* item_qkv, int D,
                      float* x, bf16* qkv, int* status, cudaStream_t st);

struct ServeAttnArgs {
  const bf16* Q; int ldq;                 // [U*C rows] candidate queries
  const bf16 *Kown, *Vown; int ldown;     // each candidate's own key / value row
  const bf16* K; int ldk; long long sk;   // cached keys of user u at K + u*sk
  const bf16* V; int ldv; long long sv;
  int U, C, nk, ns, goff, D, heads;
  const int32_t* npg;                     // [U]
  bf16* ctx; int ldc;
};
int serve_attn(const ServeAttnArgs& a, cudaStream_t st);

struct ServeHeadArgs {
  const float* x;             // [R, D] final target rows
  long long R;
  int C, D, d, hh;
  const float *cls, *ud;      // cached per user
  const float *w1, *b1, *w2, *b2;
  float* probs;               // [R]
};
void serve_head(const ServeHeadArgs& a, cudaStream_t st);

}  // namespace longer
