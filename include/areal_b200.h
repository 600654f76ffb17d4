/*
 * areal_b200.h — C-ABI of the B200-native decoupled-PPO training hot path.
 *
 * Built from paper_2505_24298_b200/csrc/ into libareal_b200.so (sm_100a).
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * passed as void*; kernels are stream-ordered and asynchronous, the library
 * never allocates device memory (callers pass workspaces) and never
 * synchronises except where noted.  No torch types cross this boundary.
 *
 * The reference (asyncrl, pure numpy) has no FFI; its drop-in boundary is the
 * Python module API of /root/reference/pkg/src/asyncrl/trainer.py.  Each entry
 * below names the reference function(s) it replaces; the Python mirror
 * paper_2505_24298_b200/trainer.py keeps the reference's names and semantics
 * on top of these calls (see INTEGRATION.md for the ctypes binding).
 *
 * Conventions
 *   - dtype codes: areal_dtype_t.  Logits/dlogits share one dtype.
 *   - per-token float arrays (behav, prox, adv, lp, entropy) are float64 and
 *     indexed by the GLOBAL token index; `row_index` (int32, may be NULL =
 *     identity) maps a logits row r to that global index, so a packed
 *     micro-batch never needs a gather pass over the per-token arrays.
 *   - status: 0 = OK, otherwise an areal_status_t; areal_status_string()
 *     gives the text.  Input validation that needs device data (allocator
 *     lengths) is reported through a device status array.
 */
#ifndef AREAL_B200_H_
#define AREAL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AREAL_ABI_VERSION 1
#define AREAL_N_STATS 8
/* Workspace every K1/K2/K3 call needs (per concurrently used stream), zeroed once
 * at allocation.  K2 uses the lower half (ticket counter, row counter + per-CTA
 * partials), K1 two more counters (its dynamic row schedule; without a workspace K1
 * falls back to a static row order), all re-armed by each launch's last CTA; K3 the
 * upper half (scratch).  One workspace must not serve two launches running
 * concurrently. */
#define AREAL_WORKSPACE_BYTES (1u << 20)
/* Largest number of sequences one minibatch may hold in the allocator. */
#define AREAL_MAX_ITEMS_PER_MINIBATCH 8192

typedef enum {
  AREAL_OK = 0,
  AREAL_ERR_INVALID_ARGUMENT = 1,
  AREAL_ERR_BAD_DTYPE = 2,
  AREAL_ERR_BAD_SHAPE = 3,
  AREAL_ERR_MISALIGNED = 4,
  AREAL_ERR_LEN_NONPOSITIVE = 5,     /* trainer.py:249-250 */
  AREAL_ERR_LEN_EXCEEDS_CAPACITY = 6,/* trainer.py:251-252 */
  AREAL_ERR_MIN_GROUPS = 7,          /* trainer.py:246-247 */
  AREAL_ERR_WORKSPACE = 8,
  AREAL_ERR_CUDA = 9,
  AREAL_ERR_UNSUPPORTED = 10,
  AREAL_ERR_BAD_CLIP_EPS = 11        /* trainer.py:48-49 */
} areal_status_t;

typedef enum { AREAL_F32 = 0, AREAL_BF16 = 1, AREAL_F16 = 2, AREAL_F64 = 3 } areal_dtype_t;

/* Kernel selection for K1/K2.  AUTO picks, for 16-byte-aligned rows of >= 16 KB:
 * K2 on 16-bit rows and on fp32 rows larger than one CTA's shared memory -> the
 * Tensor-Memory kernel (8 x 32 KB parked in TMEM, up to 7 resident in the ring, the
 * rest streamed); other K2 rows (fp32 / fp64 that fit, fp64 beyond via a cluster
 * split) and all of K1 -> ROW_RING (TMA bulk ring).  Unaligned rows of >= 16 KB:
 * K2 on 16/32-bit rows -> the TMEM kernel (masked 16-byte-aligned loads) when dlogits
 * share the logits' 16-byte phase; K1 on long rows -> the ring kernel (masked
 * 16-byte-aligned loads); otherwise one CTA per row.  Short K2 rows (<= 16 KB of
 * 16-bit, <= 32 KB of fp32 logits) -> one CTA per row, 8 per SM; other rows under
 * 16 KB (all of K1, fp64 K2) -> ROW_WARP (one warp per row).  ROW_RING /
 * ROW_WARP force the respective family. */
typedef enum { AREAL_ALGO_AUTO = 0, AREAL_ALGO_ROW_WARP = 1, AREAL_ALGO_ROW_RING = 2 } areal_algo_t;

/* Order of the float64 statistics vector (accumulated with +=). */
typedef enum {
  AREAL_STAT_OBJECTIVE_SUM = 0, /* trainer.py:188 */
  AREAL_STAT_N_VALID = 1,       /* trainer.py:191 */
  AREAL_STAT_N_CLIPPED = 2,     /* trainer.py:186, 192 */
  AREAL_STAT_RATIO_SUM = 3,     /* trainer.py:193 */
  AREAL_STAT_N_EXCLUDED = 4,    /* trainer.py:194 */
  AREAL_STAT_N_MASKED = 5,      /* extension: version-staleness / behaviour-cap mask */
  AREAL_STAT_ENTROPY_SUM = 6,   /* extension: sum of H_t over valid tokens */
  AREAL_STAT_N_TOKENS = 7
} areal_stat_t;

typedef struct {
  double clip_eps;          /* epsilon of clip(u, 1-eps, 1+eps); (0,1)           */
  double behav_weight_cap;  /* > 0: mask tokens with prox/behav weight > cap     */
  double grad_scale;        /* dlogits = grad_scale * coef * (softmax - onehot)  */
  int32_t decoupled;        /* 1: decoupled objective, 0: naive (trainer.py:165-170) */
  int32_t eta_mask;         /* >= 0: mask tokens with cur_version - version > eta */
  int32_t current_version;  /* policy version being optimised                    */
  int32_t algo;             /* areal_algo_t                                       */
  int32_t prox_from_lp;     /* 1: prox := this kernel's own lp (prox may be NULL).
                             * Valid for the first minibatch of a step, whose params
                             * are the batch-arrival params prox is defined under
                             * (trainer.py:295 vs 315-321): the prox pass and the
                             * loss then share one read of the logits, and the
                             * ratio exp(lp - prox) is exactly 1 as in the reference */
} areal_ppo_params_t;

typedef enum { AREAL_ADV_REFERENCE = 0, AREAL_ADV_GAE = 1 } areal_adv_mode_t;
typedef enum {
  AREAL_NORM_NONE = 0,
  AREAL_NORM_GLOBAL = 1,          /* token-weighted, numpy-exact (trainer.py:119-123) */
  AREAL_NORM_GROUP_TOKEN = 2,     /* GRPO, token-weighted per group                  */
  AREAL_NORM_GROUP_SEQUENCE = 3   /* GRPO, one value per trajectory                  */
} areal_norm_t;

typedef struct {
  double gamma;   /* GAE discount (reference: 1)   */
  double lam;     /* GAE lambda   (reference: 1)   */
  double eps;     /* group norm: (x - mean) / (std + eps) */
  int32_t mode;   /* areal_adv_mode_t */
  int32_t norm;   /* areal_norm_t     */
} areal_adv_params_t;

/* ---- library info ------------------------------------------------------- */
int areal_abi_version(void);
const char* areal_status_string(int status);
/* Number of stats slots a K2 launch uses in the workspace (diagnostics). */
size_t areal_workspace_bytes(void);

/* ---- kernel-selection tuning (debug / A-B API) ----------------------------
 * The shipped kernel choice is a fixed function of shapes, dtypes and
 * alignment.  These knobs override it for A/B measurement and for tests of the
 * non-default variants; nothing is read from the environment.  Values are
 * validated (AREAL_ERR_INVALID_ARGUMENT otherwise); AREAL_TUNE_DEFAULT (-1)
 * restores the shipped rule.  Process-global, read at each launch: set them
 * before launching, not concurrently with launches on other threads. */
typedef enum {
  AREAL_TUNE_K2_CLUSTER_SIZE = 0,    /* {2,4,8}: force a >= vocab split of the ring K2  */
  AREAL_TUNE_K2_TMEM = 1,            /* 0: ring/cluster K2 instead of the TMEM kernel   */
  AREAL_TUNE_K2_TMEM_STREAM = 2,     /* 0: rows beyond TMEM+ring do not stream chunks   */
  AREAL_TUNE_K2_TMEM_UNALIGNED = 3,  /* 0: unaligned rows on the row-CTA kernel         */
  AREAL_TUNE_K1_RING_UNALIGNED = 4,  /* 0: unaligned K1 rows on the row-CTA kernel      */
  AREAL_TUNE_K2_SMALL_ROWCTA_KB = 5, /* [0, 1024]: short-row kernel up to this row size */
  AREAL_TUNE_ROWCTA = 6,             /* 0: unaligned rows on the one-warp kernel        */
  AREAL_TUNE_K7_NT = 7,              /* {4,8}: K7 N-tiles per unit                      */
  AREAL_TUNE_K7_GROUP = 8,           /* [1,16]: K7 vocab blocks per token tile          */
  AREAL_TUNE_K1_CLUSTER_SIZE = 9,    /* {1,2,4,8}: K1 ring row split (default: by rows) */
  AREAL_TUNE_LMH_GROUP_M = 10,       /* [1,256]: LM-head GEMM M-tiles per raster group  */
  AREAL_TUNE_COUNT = 11
} areal_tune_t;
#define AREAL_TUNE_DEFAULT (-1)
int areal_set_tuning(int knob, int64_t value);
int areal_get_tuning(int knob, int64_t* value);

/* ---- K1: log-softmax-gather (+ entropy) ----------------------------------
 * Replaces recompute_prox_logprobs (trainer.py:128-137) ->
 * batch_token_log_probs (policy.py:159-163) -> log_softmax (policy.py:145-147)
 * on given logits.  lp_out[idx] = x_r[a] - logsumexp(x_r); entropy_out may be
 * NULL.  Reads each logits row once.
 *
 * Memory precondition (K1 and K2): rows whose start is not 16-byte aligned are
 * streamed with 16-byte bulk copies from the 16-byte boundary at or below each
 * row start to the boundary at or above its end, so the first and last row may
 * read up to 15 bytes outside [logits, logits + n_rows * ld_logits * size).  The
 * bytes are masked and never affect results; a 16-byte granule never crosses a
 * page, so the over-read cannot fault on any CUDA allocation.  Rows that start
 * on a 16-byte boundary with a 16-byte multiple length never over-read. */
int areal_logprob_fwd(const void* logits, int64_t ld_logits, int dtype, int64_t n_rows,
                      int64_t vocab, const int64_t* tokens, const int32_t* row_index,
                      double* lp_out, double* entropy_out, int algo,
                      void* workspace, size_t workspace_bytes, void* stream);

/* ---- K2: decoupled / naive PPO loss fused with its backward ---------------
 * Replaces _surrogate_terms (trainer.py:150-195) minus the model GEMMs, and
 * the per-token part of _ppo_loss (198-213).  Writes dlogits (may alias
 * logits for an in-place backward), lp/entropy per token (either may be NULL)
 * and accumulates AREAL_N_STATS float64 statistics into `stats` (device).
 * Deterministic: per-CTA partials reduced in a fixed order; the TMEM kernel (16-bit
 * rows, long fp32 rows) hands rows to CTAs dynamically and sums the objective /
 * ratio / entropy in 128-bit fixed point, so its statistics do not depend on the
 * row-to-CTA assignment either (bit-reproducible run to run). */
int areal_ppo_fwd_bwd(const void* logits, int64_t ld_logits, void* dlogits, int64_t ld_dlogits,
                      int dtype, int64_t n_rows, int64_t vocab, const int64_t* tokens,
                      const double* behav, const double* prox, const double* adv,
                      const int32_t* versions, const int32_t* row_index,
                      const areal_ppo_params_t* params, double* lp_out, double* entropy_out,
                      double* stats, void* workspace, size_t workspace_bytes, void* stream);

/* ---- K3: advantages --------------------------------------------------------
 * Replaces compute_advantages (trainer.py:114-125).  REFERENCE mode with
 * GLOBAL norm is bit-identical to the reference (numpy pairwise summation is
 * replayed).  GAE mode runs a per-sequence reverse scan (values may be NULL);
 * group norms use group_ids[n_traj] in [0, n_groups).  norm_stats_out (device,
 * 2 doubles, may be NULL) receives the global mean and std. */
int areal_advantages(const double* rewards, const int64_t* traj_bounds, int64_t n_traj,
                     int64_t n_tokens, const double* values, const int32_t* group_ids,
                     int32_t n_groups, const areal_adv_params_t* params, double* adv_out,
                     double* returns_out, double* norm_stats_out, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---- K4 + K5a: dynamic micro-batch allocation and packing plan -------------
 * Replaces allocate_microbatches (trainer.py:235-270) for M minibatches at
 * once, plus the packing order of train_step (trainer.py:310-320).
 * Items (non-empty trajectories) of minibatch m are item_traj[mb_offsets[m] ..
 * mb_offsets[m+1]) (device); their lengths come from traj_bounds.
 * Outputs (device):
 *   group_of/slot_of[n_items]    group and placement slot of each item
 *   n_groups[M]
 *   group_cu[n_items + M]        token boundaries of micro-batches in the packed
 *                                stream; minibatch m uses entries
 *                                [mb_offsets[m] + m, ... + n_groups[m]]
 *   group_seq_cu[n_items + M]    same layout, in packed-sequence units
 *   packed_traj[n_items]         trajectory id at each packed sequence position
 *   seq_cu[n_items + 1]          cu_seqlens of the whole packed stream
 *   status[M]                    0 or an areal_status_t (lengths check)
 * mb_token_start[M] (device) is the packed-stream offset of each minibatch. */
int areal_plan_microbatches(const int64_t* traj_bounds, const int32_t* item_traj,
                            const int32_t* mb_offsets, const int64_t* mb_token_start,
                            int32_t n_minibatches, int32_t n_items, int32_t max_items_per_mb,
                            int64_t capacity, int32_t min_groups, int32_t* group_of,
                            int32_t* slot_of, int32_t* n_groups, int64_t* group_cu,
                            int32_t* group_seq_cu, int32_t* packed_traj, int64_t* seq_cu,
                            int32_t* status, void* stream);

/* ---- K5b: packed gather index ----------------------------------------------
 * gather[p] = global token index of packed position p (p < seq_cu[n_items]),
 * i.e. np.concatenate([token_range(traj) for traj in packed order])
 * (trainer.py:320).  Also writes the token's packed-sequence id if seq_id is
 * non-NULL. */
int areal_fill_gather(const int64_t* traj_bounds, const int32_t* packed_traj,
                      const int64_t* seq_cu, int32_t n_items, int64_t n_packed_tokens,
                      int32_t* gather, int32_t* seq_id, void* stream);

/* ---- K7: fused LM-head GEMM + log-softmax-gather (+ entropy), tcgen05 ----------
 * Replaces recompute_prox_logprobs (trainer.py:128-137) including the model's output
 * layer: logits = features @ W.T + b (policy.py:133-142, called from
 * batch_token_log_probs, policy.py:159-163), then log_softmax (policy.py:145-147)
 * gathered at the token.  hidden [n_rows, dim] and weight [vocab, dim] are 16-bit
 * (dtype BF16 or F16, row strides ld_* in elements, multiples of 8, 16-byte aligned
 * bases); bias [vocab] fp32 or NULL; dim % 64 == 0.  Row r's global token index is
 * row_index[r] (NULL = r): lp_out[idx] = x[tok] - logsumexp(x), entropy_out (may be
 * NULL) = -sum p log p, x = hidden[r] . weight^T + bias accumulated in fp32 on the
 * tensor cores.  The [n_rows, vocab] logits never reach HBM.  scratch (device) holds
 * per-(row, vocab block, column half) partials: areal_linear_logprob_scratch_bytes()
 * (sized for the smallest vocab block, 1024 columns; 32 B per row per block).
 * cta_group: 1 = one CTA per 128-token tile (tcgen05 .cta_group::1, M=128),
 * 2 = a CTA pair per 256-token tile (.cta_group::2, M=256, each CTA loads half of the
 * W tile), 0 = choose (2 when n_rows > 128). */
size_t areal_linear_logprob_scratch_bytes(int64_t n_rows, int64_t vocab);
int areal_linear_logprob_fwd(const void* hidden, int64_t ld_hidden, const void* weight,
                             int64_t ld_weight, const float* bias, int dtype, int64_t n_rows,
                             int64_t vocab, int64_t dim, const int64_t* tokens,
                             const int32_t* row_index, double* lp_out, double* entropy_out,
                             void* scratch, size_t scratch_bytes, int cta_group, void* stream);

/* ---- LM-head GEMMs of the loss + backward (tcgen05) -------------------------
 * The model side of _surrogate_terms (trainer.py:163, 183-184): logits =
 * features W^T + b, grad_w = resid^T features, grad_b = sum(resid), for an LM head
 * W [V, d] over hidden states H [T, d] (16-bit; fp32 accumulation in TMEM).  With
 * K2 turning a logits chunk into dlogits dL in place, one micro-batch chunk is
 *   AREAL_LMH_LOGITS   C[M=T, N=V] (16-bit) = A[T, d] B[V, d]^T + bias[V]   (K = d)
 *   AREAL_LMH_DHIDDEN  C[M=T, N=d] (16-bit) = A[T, V] B[V, d]               (K = V)
 *   AREAL_LMH_DWEIGHT  C[M=V, N=d] (fp32, += if accumulate) = A[T, V]^T B[T, d]
 *                                                                           (K = T)
 * (row-major operands with row strides lda / ldb / ldc elements, 16-byte aligned,
 * strides multiples of 16 bytes; bias fp32 [N] or NULL, LOGITS only), and
 * areal_colsum gives grad_b (+)= column sums of dL.  dtype: AREAL_BF16 / AREAL_F16
 * for A, B and the 16-bit outputs.  Stream-ordered; no allocation. */
typedef enum { AREAL_LMH_LOGITS = 0, AREAL_LMH_DHIDDEN = 1, AREAL_LMH_DWEIGHT = 2 } areal_lmh_op_t;
int areal_lm_head_gemm(int op, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                       int64_t ldc, int64_t M, int64_t N, int64_t K, const float* bias,
                       int accumulate, int dtype, void* stream);
/* The chunk's whole backward through the head in ONE launch (grouped GEMM: the
 * DHIDDEN units, then the DWEIGHT units filling the first's last wave), with grad_b
 * summed from the dlogits tiles while DWEIGHT holds them in shared memory:
 *   grad_hidden[n_rows, dim] (16-bit)  = dL[n_rows, vocab] W[vocab, dim]
 *   grad_weight[vocab, dim] (fp32)    (+)= dL^T hidden[n_rows, dim]
 *   grad_bias[vocab] (fp32, may be NULL) (+)= sum_r dL[r, :]
 * (+= when accumulate; deterministic).  trainer.py:183-184. */
int areal_lm_head_backward(const void* dlogits, int64_t ld_dlogits, const void* hidden,
                           int64_t ld_hidden, const void* weight, int64_t ld_weight,
                           int64_t n_rows, int64_t vocab, int64_t dim, void* grad_hidden,
                           int64_t ld_grad_hidden, float* grad_weight, int64_t ld_grad_weight,
                           float* grad_bias, int accumulate, int dtype, void* stream);
/* out[c] (+)= sum_r x[r, c] in fp32, deterministic (fixed-order block partials in
 * `scratch`, areal_colsum_scratch_bytes(rows, cols) bytes). */
size_t areal_colsum_scratch_bytes(int64_t rows, int64_t cols);
int areal_colsum(const void* x, int64_t ld, int64_t rows, int64_t cols, int dtype, float* out,
                 int accumulate, void* scratch, size_t scratch_bytes, void* stream);

/* ---- behaviour log-prob recording at emission ------------------------------
 * Replaces the per-token record of RolloutWorker.step (rollout.py:154-159:
 * tokens.append(token); behavior_logprobs.append(P.log_prob(params, features,
 * token)); versions.append(params.version)) for one decode step of n_rows live
 * sequences.  Row r belongs to slot slots[r] (distinct within a step); its token
 * and *version (device int32: graph-capturable) are appended at position lengths[slot]++ of that slot's row in
 * tok_buf / ver_buf ([n_slots * max_len + 1]; the last entry is a sink), and
 * row_index_out[r] receives the flat position, so a following
 * areal_logprob_fwd / areal_linear_logprob_fwd(tokens = tok_buf, row_index =
 * row_index_out, lp_out = lp_buf) writes the log-prob beside them.  A bad slot
 * or a full slot sends the row to the sink and raises *status (device int32,
 * atomicMax of AREAL_ERR_BAD_SHAPE / AREAL_ERR_LEN_EXCEEDS_CAPACITY). */
int areal_emission_append(const int32_t* slots, const int64_t* step_tokens, int64_t n_rows,
                          const int32_t* version, int32_t n_slots, int64_t max_len, int32_t* lengths,
                          int64_t* tok_buf, int32_t* ver_buf, int32_t* row_index_out,
                          int32_t* status, void* stream);

/* ---- K6: fused global-norm clip + Adam (decoupled weight decay), multi-tensor --
 * Replaces the optimizer step of train_step (trainer.py:329-331): grad.scale_(-1/n)
 * then apply_update (policy.py:225-258) with clip_by_global_norm (policy.py:215-221).
 * For every tensor k (n_tensors <= AREAL_ADAM_MAX_TENSORS):
 *   g = grad*grad_scale; norm = sqrt(sum_k sum(g_k**2)); if clip_norm > 0 and
 *   norm > clip_norm: g *= clip_norm/norm; m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g;
 *   p -= lr*((m/c1)/(sqrt(v/c2) + eps) + wd*p).
 * The host passes the scalars the reference computes in Python ((1-b), c = 1-b**step,
 * grad_scale = -1/n).  exact_norm = 1 (fp64 only) replays numpy's pairwise sums so the
 * update is bit-identical to the reference for the same gradient.  If any scaled
 * gradient is non-finite nothing is written and norm_out[1] (device, may be NULL;
 * norm_out[0] = global norm) counts them: the caller raises NonFiniteGradientError
 * (policy.py:234-239).  param/exp_avg/exp_avg_sq share param_dtype (F64 or F32);
 * grads are F64 with F64 params, or F32/BF16/F16 with F32 master params.  No host
 * synchronisation.  Uses the upper half of the workspace (like K3). */
#define AREAL_ADAM_MAX_TENSORS 32

typedef struct {
  void* param;
  const void* grad;
  void* exp_avg;
  void* exp_avg_sq;
  int64_t numel;
} areal_adam_tensor_t;

typedef struct {
  double lr, beta1, beta2, eps, weight_decay, clip_norm; /* AdamConfig (policy.py:188-196) */
  double one_minus_beta1, one_minus_beta2;               /* 1 - beta, as Python computes it */
  double bias_correction1, bias_correction2;             /* 1 - beta**step (policy.py:249-250) */
  double grad_scale;                                     /* -1/n (trainer.py:330) or 1 */
  int32_t exact_norm;                                    /* 1: numpy-exact fp64 norm */
  /* optional DEVICE pointer: if set, the scale is grad_scale / max(*grad_scale_divisor, 1)
   * computed on the device — e.g. grad_scale = -1 and the divisor = the all-reduced
   * n_valid statistic of K2 (stats[1]), i.e. trainer.py:329-330's -1/max(n,1) with no
   * host synchronisation between the loss and the optimizer step */
  const double* grad_scale_divisor;
} areal_adam_params_t;

int areal_adam_step(const areal_adam_tensor_t* tensors, int32_t n_tensors, int param_dtype,
                    int grad_dtype, const areal_adam_params_t* params, double* norm_out,
                    void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AREAL_B200_H_ */
