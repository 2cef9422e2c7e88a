/* rf_oracle.h — TEST INFRASTRUCTURE ONLY (see rf_oracle.c header).
 * fp64 restatement of the reference loss path on the packed LLM layout of
 * include/rf_offpolicy.h; all arrays are host fp64/int arrays. */
#ifndef RF_ORACLE_H
#define RF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t variant, aggregation;
    double clip_eps, eps_low, eps_high, trunc_cap, kl_weight, w_plus, w_minus, engine_mismatch_cap;
} rfo_config; /* = rlsim::LossConfig, losses.hpp:28-41 */

typedef struct {
    int64_t num_tokens, num_seqs;
    int32_t vocab, normalization; /* 0 = SEQ_THEN_BATCH (reference), 1 = GLOBAL_TOKEN */
    const double* logits;         /* rows of V doubles */
    int64_t row_stride;
    const int32_t* row_of_token;  /* NULL -> row t */
    const double* ref_logits;     /* KL rows, same row indexing */
    int64_t ref_row_stride;
    const int32_t* token_ids;
    const int64_t* seq_offsets;   /* [N+1]; token t of this call = seq_offsets[0] + local index */
    const double* advantages;     /* [N] */
    const double* behavior_logp, *prox_logp, *engine_logp; /* [T] */
    int64_t global_num_seqs, global_num_tokens;
    double grad_sign;
} rfo_batch;

typedef struct {
    double* dlogits; /* [T x dlogits_row_stride] per-token rows or NULL */
    int64_t dlogits_row_stride;
    double *token_logp, *token_ratio, *token_coef, *token_loss;
    uint8_t* token_flags;
    double* value;
} rfo_outputs;

int rfo_validate(const rfo_config* c);
void rfo_log_softmax(const double* row, int32_t V, double* out);
int rfo_grpo_advantages(const double* rewards, const int64_t* group_offsets, int64_t num_groups, double* adv,
                        uint8_t* degenerate);
int rfo_loss_and_grad(const rfo_config* c, const rfo_batch* b, rfo_outputs* o);

#ifdef __cplusplus
}
#endif
#endif
