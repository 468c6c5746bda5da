/* longer.h — C ABI of the B200 (sm_100a) LONGER encoder library `_longer_sm100.so`.
 *
 * The reference (`longrec`, pure Python/NumPy) has no FFI layer; its seam is the module API
 * (SURVEY.md §8b).  These entry points replace, for a whole batch at once:
 *
 *   longer_forward           LongRecModel.forward_tensor over a batch + sigmoid
 *                            (pkg/src/longrec/model.py:307-363, :365-377)
 *   longer_forward_backward  the train-step body: zero_grads → per-sample T.bce(forward_tensor)
 *                            → T.mean_scalars → loss.backward() (pkg/src/longrec/model.py:555-567;
 *                            pkg/src/longrec/tensors.py:536-571, :141-175)
 *   longer_adam_step         Adam.step (pkg/src/longrec/model.py:453-482)
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every buffer is allocated by the caller (device memory,
 *     stream-ordered); the library never allocates global memory.
 *   - `params` / `grads` are ONE contiguous fp32 array each, holding every parameter in the
 *     reference `LongRecModel.params()` order and shapes (row-major, weights [in, out]);
 *     `longer_param_count` gives its length.
 *   - `ws` is scratch of at least `longer_workspace_bytes` bytes (256-byte aligned).
 *   - Return value: 0 on success, otherwise a LONGER_E* code; `longer_last_error()` gives text.
 *     Codes map 1:1 onto the reference exception classes (pkg/src/longrec/errors.py:8-29).
 *   - Calls are stream-ordered and graph-capturable (no host synchronisation inside) and
 *     re-entrant: all per-call state lives in `ws` or on the stack; the only process-wide state
 *     is the per-(kernel, device) shared-memory attribute cache.  The weight-gradient side
 *     stream, its fork/join events, the LONGER_* tuning switches (read at every call) and the
 *     diagnostic probes are per calling thread, so two threads may drive two models (or two
 *     devices) concurrently, each with its own workspace.
 */
#ifndef LONGER_H_
#define LONGER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LONGER_OK 0
#define LONGER_ECONFIG 1      /* ConfigError */
#define LONGER_EDIM 2         /* DimensionError */
#define LONGER_ELOOKUP 3      /* EmbeddingLookupError */
#define LONGER_ENUMERIC 4     /* NumericalError */
#define LONGER_ESTALE 5       /* StaleCacheError */
#define LONGER_ECUDA 6        /* CUDA runtime failure (RuntimeError) */

/* ModelConfig fields (pkg/src/longrec/config.py:29-49) + batch size. */
typedef struct LongerDims {
  int32_t L, d, K, m, k, N, heads;
  int32_t merge_inner;      /* 0 = "concat", 1 = "inner" */
  int32_t inner_layers;
  int32_t query_strategy;   /* 0 recent, 1 uniform, 2 learnable, 3 recent_uniform (config.py order) */
  int32_t head_hidden, d_item, d_act, d_time, n_time_buckets;
  int32_t vocab, n_actions, n_users, n_profiles;
  int32_t batch;            /* samples in this call */
} LongerDims;

/* A batch in the right-aligned layout of encode_events (pkg/src/longrec/inputs.py:457-482):
 * sample b's n_events[b] real events occupy token columns L-n .. L-1. Device pointers. */
typedef struct LongerBatch {
  const int32_t* items;     /* [B, L] */
  const int32_t* actions;   /* [B, L] */
  const int32_t* dt;        /* [B, L] candidate_ts - event_ts (>= 0, seconds) */
  const int32_t* n_events;  /* [B] */
  const int32_t* uid;       /* [B] */
  const int32_t* profile;   /* [B] */
  const int32_t* cand_item; /* [B] */
  const float* label;       /* [B] 0/1 */
} LongerBatch;

int longer_param_count(const LongerDims* dims, int64_t* count);
int longer_workspace_bytes(const LongerDims* dims, size_t* bytes);

/* probs[B] = sigmoid(logit).  Inference: no activations are kept for backward. */
int longer_forward(const LongerDims* dims, const float* params, const LongerBatch* batch,
                   void* ws, size_t ws_bytes, float* probs, void* stream);

/* Activation trace of a forward (the reference's ForwardTrace, pkg/src/longrec/model.py:129-143,
 * :365-372): device pointers into `ws`, valid until the next call on the same workspace. */
typedef struct LongerTrace {
  const float* h;              /* [B, Lp, d] token-MLP output, left zero rows for pad events */
  const float* merged;         /* [B, G, D] merged sequence (InnerTrans / concat) */
  const int32_t* query_groups; /* [B, k] merged group of each sequence query; null: "recent"
                                  (G-k+i) or "learnable" (bank rows, no group) */
  const float* layers[17];     /* [B, q, D] output of the cross block, then of each self block */
  const float* head_input;     /* [B, head_width] [t, c, t*c, t*t, uid_emb, profile_emb] */
  int32_t n_layers, Lp, G, q, head_width;
} LongerTrace;

/* longer_forward that also keeps every row of every layer and returns where the activations are. */
int longer_forward_trace(const LongerDims* dims, const float* params, const LongerBatch* batch,
                         void* ws, size_t ws_bytes, float* probs, LongerTrace* trace, void* stream);

/* Training step body: probs[B], loss[0] = batch-mean BCE, grads (overwritten) = dloss/dparams. */
int longer_forward_backward(const LongerDims* dims, const float* params, const LongerBatch* batch,
                            void* ws, size_t ws_bytes, float* probs, float* loss, float* grads,
                            void* stream);

/* Vector-Jacobian product of the most recent longer_forward on the same ws / batch / params (the
 * torch.autograd bridge): grads (overwritten) = (dprobs/dparams)ᵀ · dprobs, using the
 * activations that forward left in `ws`. */
int longer_backward(const LongerDims* dims, const float* params, const LongerBatch* batch, void* ws,
                    size_t ws_bytes, const float* probs, const float* dprobs, float* grads, void* stream);

/* In-place Adam on the flat buffers (beta1 .9, beta2 .999, eps 1e-8, bias-corrected, step t>=1).
 * m, v: fp32 [count] moments (caller-zeroed before step 1). */
int longer_adam_step(float* params, const float* grads, float* m, float* v, int64_t count, float lr,
                     int32_t t, void* stream);

/* Device-side input validation flags accumulated since the last call (and reset):
 * bit0 = id out of range (EmbeddingLookupError), bit1 = negative time delta (ConfigError).
 * Reads back through a synchronous copy on `stream`. */
int longer_read_status(void* ws, int32_t* flags, void* stream);

const char* longer_last_error(void);

/* ---- Two-stage serving (pkg/src/longrec/serving.py:84-167) --------------------------------
 * Stage 1, `longer_cache_build`, replaces build_cache (serving.py:84-144) for `dims->batch` users
 * at once: the batch carries each user's events with dt measured from that user's scoring time
 * (cand_item and label are ignored and may be null).  It stores, per user, everything that does
 * not depend on the candidate: the cross layer's key/value rows of the merged sequence and the
 * m-1 non-target globals, each self layer's key/value rows of the k+m-1 non-target queries
 * (bf16, the exact rows the full forward feeds its attention), the last layer's CLS row and the
 * user-side head features.  `cache` is caller-owned device memory of `longer_cache_bytes`.
 * Stage 2, `longer_cache_score`, replaces score_with_cache (serving.py:147-167) for
 * `candidates_per_user` candidates of every cached user (cand_items[u * C + j], probs likewise):
 * only the target rows run through the blocks, against the cached rows plus their own key/value.
 * Fingerprint / scoring-time staleness (StaleCacheError) is tracked by the host wrapper; the
 * library checks that the cache size matches `dims` (LONGER_ESTALE otherwise). */
int longer_cache_bytes(const LongerDims* dims, size_t* bytes);
int longer_cache_build(const LongerDims* dims, const float* params, const LongerBatch* batch,
                       void* ws, size_t ws_bytes, void* cache, size_t cache_bytes, void* stream);
int longer_score_workspace_bytes(const LongerDims* dims, int32_t candidates_per_user, size_t* bytes);
int longer_cache_score(const LongerDims* dims, const float* params, const void* cache,
                       size_t cache_bytes, const int32_t* cand_items, int32_t candidates_per_user,
                       void* ws, size_t ws_bytes, float* probs, void* stream);

/* Overlapped data-parallel gradient reduction.  grads[early_begin, count) — the
 * cross and self blocks, the query bank and the head, about 2/3 of the parameters — are final
 * before the front-end backward starts.  With an event set (caller-owned cudaEvent_t, per calling
 * thread; null disables), longer_forward_backward / longer_backward record it at that point, on a
 * stream that has joined all prior work of the call, so a communication stream can wait on it and
 * reduce that range while the front-end backward runs; the rest is final when the call's stream
 * reaches the end of the call. */
int longer_grad_early_begin(const LongerDims* dims, int64_t* begin);
int longer_set_grad_event(void* ev);

/* Diagnostics: record caller-owned CUDA events (cudaEvent_t) immediately before / after one fused
 * kernel of subsequent calls, on the call's stream (graph-capturable).  phase: 0 front-end forward,
 * 1 InnerTrans backward, 2 token-MLP/featuriser backward, 3 cross-attention forward,
 * 4 cross-attention backward; sections: 5 forward after the front-end (globals, blocks, head),
 * 6 backward before the front-end (head, blocks, globals).  Null events disable the probe. */
int longer_set_probe(int32_t phase, void* ev_begin, void* ev_end);

#ifdef __cplusplus
}
#endif
#endif /* LONGER_H_ */
