/*
 * rf_offpolicy.h — C ABI of the B200-native off-policy loss + dlogits hot path.
 *
 * Drop-in boundary for the reference's loss library (rlsim, C++20):
 *
 *   rlsim::LossResult rlsim::loss_and_grad(const LossConfig&, const ToyPolicy&,
 *                                          const std::vector<Trajectory>&,
 *                                          const LossInputs& = {});
 *       -> /root/reference/proj/include/rlsim/losses.hpp:77-78, proj/src/losses.cpp:137-331
 *   rlsim::GroupAdvantages rlsim::grpo_advantages(const std::vector<double>&);
 *       -> losses.hpp:50, losses.cpp:41-60
 *   rlsim::LossConfig / LossConfig::validate / LossVariant / to_string / loss_variant_from_string
 *       -> losses.hpp:10-41, losses.cpp:8-39
 *
 * The reference takes a tabular fp64 policy [contexts x vocab] and a vector of
 * Trajectory records (policy.hpp:44-51).  The ABI takes the LLM-native packed
 * layout instead — a [rows x vocab] logits matrix (bf16 or f32), one row per
 * token (row_of_token == NULL) or rows shared per context (row_of_token given,
 * "mapping B"), and CSR-packed ragged sequences.  Each reference Trajectory
 * maps to one sequence; each Trajectory::context maps to the row every token of
 * that sequence reads.  See DESIGN.md §2 for the full mapping.
 *
 * Conventions
 *   - All pointers in rf_batch / rf_outputs passed to rf_loss_and_grad and
 *     rf_grpo_advantages are DEVICE pointers; the calls are stream-ordered and
 *     asynchronous, hold no global state and are reentrant per stream.
 *   - Host-detectable errors (the reference's std::invalid_argument throw sites)
 *     return synchronously as rf_status.  Device-detected errors (non-finite
 *     ratio, losses.cpp:205,267; token id out of range) are OR-ed into
 *     *outputs->device_status (RF_DEVSTAT_* bits) — read it after a sync.
 *   - Sign: the reference returns the objective J (to MAXIMISE) and dJ/dlogits
 *     (losses.hpp:74-78).  grad_sign = +1 reproduces that; -1 gives d(-J).
 *   - rf_loss_and_grad ACCUMULATES into outputs->scalars (so a batch can be
 *     streamed in token chunks); zero them with rf_zero_scalars first.
 */
#ifndef RF_OFFPOLICY_H
#define RF_OFFPOLICY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Ordinals equal rlsim::LossVariant (losses.hpp:10-18). */
typedef enum {
    RF_PPO = 0,
    RF_DECOUPLED_PPO = 1,
    RF_TIS = 2,
    RF_CISPO = 3,
    RF_TOPR = 4,
    RF_GRPO = 5,
    RF_NAIVE_IS = 6
} rf_loss_variant;

/* Ordinals equal rlsim::RatioAggregation (losses.hpp:23-26). */
typedef enum { RF_TOKEN_MEAN = 0, RF_SEQUENCE_PRODUCT = 1 } rf_ratio_aggregation;

/* Token weight normalisation.
 *   SEQ_THEN_BATCH: 1/(N_global * L_i) per token (token_mean) and 1/N_global per
 *                   sequence (sequence_product) — the reference's inv_n/len
 *                   (losses.cpp:152,167).
 *   GLOBAL_TOKEN:   1/T_global per token — the LLM "token-mean over the global
 *                   batch"; identical to the reference run on length-1
 *                   trajectories (one per token, "mapping A"). */
typedef enum { RF_NORM_SEQ_THEN_BATCH = 0, RF_NORM_GLOBAL_TOKEN = 1 } rf_normalization;

typedef enum { RF_DTYPE_BF16 = 0, RF_DTYPE_F32 = 1, RF_DTYPE_F64 = 2 } rf_dtype;

typedef enum {
    RF_OK = 0,
    /* LossConfig::validate, losses.cpp:33-38 (one code per throw). */
    RF_ERR_CLIP_EPS = 1,
    RF_ERR_EPS_LOW_HIGH = 2,
    RF_ERR_TRUNC_CAP = 3,
    RF_ERR_KL_WEIGHT = 4,
    RF_ERR_TOPR_WEIGHTS = 5,
    RF_ERR_MISMATCH_CAP = 6,
    /* loss_and_grad / grpo_advantages throw sites. */
    RF_ERR_EMPTY_BATCH = 7,          /* losses.cpp:140 */
    RF_ERR_MISSING_PROX = 8,         /* losses.cpp:142-144 */
    RF_ERR_MISSING_REF = 9,          /* losses.cpp:145-148 */
    RF_ERR_EMPTY_TRAJECTORY = 10,    /* losses.cpp:157 */
    RF_ERR_MISSING_ENGINE_LOGP = 11, /* losses.cpp:173-174,194-196 */
    RF_ERR_NONFINITE_RATIO = 12,     /* losses.cpp:205,267 (device-detected) */
    RF_ERR_GROUP_TOO_SMALL = 13,     /* losses.cpp:42 */
    RF_ERR_UNKNOWN_VARIANT = 14,     /* losses.cpp:29 */
    /* ABI-level validation the reference leaves as UB. */
    RF_ERR_INVALID_ARGUMENT = 15,
    RF_ERR_UNSUPPORTED_LAYOUT = 16,
    RF_ERR_TOKEN_OUT_OF_RANGE = 17,
    RF_ERR_WORKSPACE_TOO_SMALL = 18,
    RF_ERR_CUDA = 19
} rf_status;

/* Bits of *device_status. */
#define RF_DEVSTAT_NONFINITE_RATIO 0x1    /* exp(lp - b) not finite (losses.cpp:205,267) */
#define RF_DEVSTAT_TOKEN_OUT_OF_RANGE 0x2 /* token id outside [0, V) (UB in the reference) */
#define RF_DEVSTAT_GROUP_TOO_SMALL 0x4    /* rf_grpo_advantages: a group of < 2 (losses.cpp:42);
                                             its advantages are zeroed */
#define RF_DEVSTAT_EMPTY_TRAJECTORY 0x8   /* a sequence with no tokens (losses.cpp:157), checked
                                             over the sequences each call spans */

/* Per-token flag bits (token_flags[t]).  Bit-exact contract vs the reference's
 * branch conditions (losses.cpp:275-312):
 *   CLIPPED     ppo/grpo: r*A > clip(r)*A   (gradient zeroed, losses.cpp:275-280)
 *               decoupled_ppo: r*A > po*c*A and tp != c   (losses.cpp:283-290)
 *               tis / cispo: r_sg outside [lo, hi]          (losses.cpp:294,305)
 *               topr: A <= 0 and r_sg outside [0, cap]      (losses.cpp:311-312)
 *   TOPR_POS    topr: A > 0 (T+ set)
 *   MISMATCH_CAPPED  cap > 0 and exp(b - e) > cap           (losses.cpp:170-176)
 *   NONFINITE   exp(lp - b) not finite (the reference throws)
 *   ZERO_COEF   dlogits row coefficient is exactly 0 (row left at +0.0, losses.cpp:103) */
#define RF_FLAG_CLIPPED 0x01
#define RF_FLAG_TOPR_POS 0x02
#define RF_FLAG_MISMATCH_CAPPED 0x04
#define RF_FLAG_NONFINITE 0x08
#define RF_FLAG_ZERO_COEF 0x10

/* scalars[] layout (fp64, accumulated). */
#define RF_SCALAR_LOSS 0      /* objective J (sign per reference: maximised) */
#define RF_SCALAR_TOKENS 1    /* tokens processed */
#define RF_SCALAR_CLIPPED 2   /* tokens with RF_FLAG_CLIPPED */
#define RF_SCALAR_NONFINITE 3 /* tokens with RF_FLAG_NONFINITE */
#define RF_SCALAR_ZERO_COEF 4 /* tokens with RF_FLAG_ZERO_COEF */
#define RF_SCALAR_MISMATCH 5  /* tokens with RF_FLAG_MISMATCH_CAPPED */
#define RF_SCALAR_KL 6        /* sum of scale * KL (grpo with kl_weight > 0) */
#define RF_SCALAR_COEF_ABS 7  /* sum |coef| (diagnostic) */
#define RF_NUM_SCALARS 8

/* = rlsim::LossConfig (losses.hpp:28-41). */
typedef struct {
    int32_t variant;     /* rf_loss_variant */
    int32_t aggregation; /* rf_ratio_aggregation */
    double clip_eps;
    double eps_low;
    double eps_high;
    double trunc_cap;
    double kl_weight;
    double w_plus;
    double w_minus;
    double engine_mismatch_cap;
} rf_loss_config;

/* A packed ragged batch (or a token chunk of one; see rf_loss_and_grad). */
typedef struct {
    int64_t num_tokens; /* T (tokens in this call) */
    int64_t num_seqs;   /* N (length of seq_offsets - 1, advantages, rewards) */
    int64_t num_groups; /* GRPO groups (rf_grpo_advantages) */
    int32_t vocab;      /* V */
    int32_t logits_dtype;       /* RF_DTYPE_BF16 | RF_DTYPE_F32 */
    const void* logits;         /* rows of V logits */
    int64_t logits_row_stride;  /* elements between rows */
    const int32_t* row_of_token; /* [T] row per token; NULL -> row t */
    const int32_t* token_ids;    /* [T] sampled token ids */
    const int32_t* seq_of_token; /* [T] sequence index of each token (into seq arrays) */
    const int64_t* seq_offsets;  /* [N+1] CSR token offsets (global token index space) */
    const int64_t* group_offsets; /* [num_groups+1] CSR over sequences (GRPO groups) */
    const double* rewards;       /* [N] (rf_grpo_advantages input) */
    const double* advantages;    /* [N] per-sequence advantage (rf_loss_and_grad input) */
    int32_t logp_dtype;          /* RF_DTYPE_F32 | RF_DTYPE_F64 for the three arrays below */
    int32_t normalization;       /* rf_normalization */
    const void* behavior_logp;   /* [T] Trajectory::behavior_logp */
    const void* prox_logp;       /* [T] proximal-policy log-prob of the token (decoupled_ppo) */
    const void* engine_logp;     /* [T] Trajectory::engine_logp (engine_mismatch_cap > 0) */
    const void* ref_logits;      /* reference-policy rows (grpo with kl_weight > 0), same
                                    dtype/row indexing as logits */
    int64_t ref_row_stride;
    int64_t global_num_seqs;     /* N_global for SEQ_THEN_BATCH (sum over shards/chunks) */
    int64_t global_num_tokens;   /* T_global for GLOBAL_TOKEN */
    double grad_sign;            /* +1: dJ/dlogits (reference); -1: d(-J)/dlogits */
} rf_batch;

typedef struct {
    void* dlogits;               /* [T rows] per-token dlogits; NULL = do not write */
    int32_t dlogits_dtype;       /* RF_DTYPE_BF16 | RF_DTYPE_F32 */
    int32_t _pad0;
    int64_t dlogits_row_stride;  /* elements */
    double* token_logp;          /* [T] log pi(token) (optional) */
    double* token_ratio;         /* [T] exp(lp - behavior) (optional) */
    double* token_coef;          /* [T] dlogits row coefficient k_t (optional) */
    double* token_loss;          /* [T] contribution to J (optional) */
    uint8_t* token_flags;        /* [T] RF_FLAG_* (optional) */
    double* advantages_out;      /* [N] rf_grpo_advantages output */
    uint8_t* group_degenerate;   /* [num_groups] rf_grpo_advantages output */
    double* scalars;             /* [RF_NUM_SCALARS] accumulated (required) */
    int32_t* device_status;      /* [1] RF_DEVSTAT_* bits (required) */
    void* workspace;             /* device scratch of rf_workspace_bytes() */
    size_t workspace_bytes;
} rf_outputs;

/* Kernel selection (for tests and benchmarks). AUTO picks the cluster/TMA ring
 * kernel when the row layout allows it, else the generic kernel. */
typedef enum { RF_KERNEL_AUTO = 0, RF_KERNEL_RING = 1, RF_KERNEL_GENERIC = 2 } rf_kernel;

/* ---- registry (losses.cpp:8-39) ---- */
void rf_loss_config_default(rf_loss_config* cfg);           /* losses.hpp:28-38 defaults */
rf_status rf_loss_config_validate(const rf_loss_config* cfg);
const char* rf_loss_variant_name(int32_t variant);          /* to_string; "unknown" */
rf_status rf_loss_variant_from_name(const char* name, int32_t* variant_out);
const char* rf_status_string(rf_status status);

/* ---- device API (stream-ordered; all buffers device-resident) ---- */
/* Scratch for one call: 64 bytes per token (one fp64 partial-scalar row per token,
 * reduced in a fixed order), the row counters, and for sequence_product / exact KL
 * their per-token and exchange arrays. */
size_t rf_workspace_bytes(const rf_loss_config* cfg, const rf_batch* batch);

/* K1: GRPO group-relative advantages (grpo_advantages, losses.cpp:41-60), one
 * group per CSR segment of batch->group_offsets over batch->rewards.  Writes
 * outputs->advantages_out[N] and outputs->group_degenerate[num_groups]. */
rf_status rf_grpo_advantages(const rf_batch* batch, rf_outputs* outputs, void* stream);

rf_status rf_zero_scalars(rf_outputs* outputs, void* stream);

/* K2(+K3): per-token log-softmax/gather, importance ratio, surrogate value and
 * dlogits in one pass over the logits (loss_and_grad, losses.cpp:137-331). */
rf_status rf_loss_and_grad(const rf_loss_config* cfg, const rf_batch* batch, rf_outputs* outputs,
                           void* stream);
rf_status rf_loss_and_grad_ex(const rf_loss_config* cfg, const rf_batch* batch, rf_outputs* outputs,
                              void* stream, int32_t kernel);

/* Segmented row sums for the reference-layout gradient: for every segment s,
 *   out[s * out_stride + v] = sum over i in [seg_offsets[s], seg_offsets[s+1]) of
 *                             rows[seg_rows[i] * row_stride + v]      (v < width)
 * in fp64, in index order (deterministic).  With rows = per-token dlogits and one
 * segment per context listing that context's tokens, this is LossResult.grad
 * (LogProbGrad's per-context accumulation, losses.cpp:87-115).  Device pointers,
 * stream-ordered; rows bf16 or f32; at most 65,535 segments per call. */
rf_status rf_rows_segment_sum(const void* rows, int32_t rows_dtype, int64_t row_stride, const int64_t* seg_offsets,
                              const int32_t* seg_rows, int64_t num_segments, int32_t width, double* out,
                              int64_t out_stride, void* stream);

/* Number of CUDA kernel launches the last rf_loss_and_grad* call made on this
 * thread (for benchmark accounting). */
int32_t rf_last_launch_count(void);

/* Profiling aid: per-phase cycle counters of the fused kernel, accumulated when
 * the process runs with RF_DEBUG_COUNTERS=1 (else returns 0).  Synchronises the
 * device; copies up to n counters into out and optionally resets them.  Words
 * 0..15 are the phase counters; from word 16 the profiling build stores each
 * CTA's consumer start / end time (%globaltimer ns), two words per CTA. */
int32_t rf_debug_counters(uint64_t* out, int32_t n, int32_t reset);

/* ---- experimental: the step before ----
 * LM-head GEMM on the tensor cores (tcgen05) with the softmax statistics fused into
 * its epilogue: for hidden states H [T, K] and the vocab projection W [V, K] (both
 * bf16, row-major, K a multiple of 64, rows 16-byte aligned), writes
 * lse[t] = log Σ_v exp((H Wᵀ)[t, v]) (fp64) and x_tok[t] = (H Wᵀ)[t, token_ids[t]] (fp32)
 * without materialising the [T, V] logits.  Device pointers, stream-ordered.
 * No reference counterpart: the reference's policy is a logits table
 * (policy.hpp ToyPolicy::logits); this is the fusion §8(f) names next. */
rf_status rf_lmhead_lse(const void* hidden, const void* w_vocab, const int32_t* token_ids, int64_t num_tokens,
                        int32_t vocab, int32_t hidden_dim, double* lse, float* x_tok, void* stream);

/* The dlogits half: recomputes the logits tiles on the tensor cores and writes
 * dlogits[t, v] = coef[t]·(1[v = token_ids[t]] − exp((H Wᵀ)[t, v] − lse[t])) as bf16 rows
 * of stride dlogits_row_stride (16-byte aligned rows), lse from rf_lmhead_lse and coef
 * the per-token loss coefficient (rf_outputs.token_coef of the loss math). */
rf_status rf_lmhead_dlogits(const void* hidden, const void* w_vocab, const int32_t* token_ids, int64_t num_tokens,
                            int32_t vocab, int32_t hidden_dim, const double* lse, const double* coef, void* dlogits,
                            int64_t dlogits_row_stride, void* stream);

/* The per-token loss math between the two LM-head sweeps: lp = x_tok − lse, then the
 * surrogate, coefficient, clip flags and scalars of rf_loss_and_grad (token_mean
 * aggregation, no exact KL; batch->logits is not read).  outputs->token_coef feeds
 * rf_lmhead_dlogits; outputs->scalars accumulates like rf_loss_and_grad. */
rf_status rf_token_loss_from_stats(const rf_loss_config* cfg, const rf_batch* batch, const double* lse,
                                   const float* x_tok, rf_outputs* outputs, void* stream);

/* ---- host API: the reference-facing call with HOST buffers ----
 * Same semantics as rf_loss_and_grad but every pointer in batch/outputs is a
 * host pointer (pinned memory recommended).  Streams the batch through the GPU
 * in token chunks on `device`, overlapping H2D of chunk i+1, compute of chunk
 * i and D2H of chunk i-1's dlogits.  Synchronous: returns after the scalars
 * and every requested output are back on the host. */
rf_status rf_loss_and_grad_host(const rf_loss_config* cfg, const rf_batch* batch, rf_outputs* outputs,
                                int32_t device, int64_t chunk_tokens);

#ifdef __cplusplus
}
#endif

#endif /* RF_OFFPOLICY_H */
