/*
 * rf_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64, single-threaded restatement of the reference's off-policy
 * loss path (rlsim, /root/reference/proj/src/losses.cpp + policy.cpp), written
 * directly against the LLM-packed layout of include/rf_offpolicy.h.  It is the
 * CHECKER for the CUDA path: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * (paper_2510_11345_b200/) never links or calls it.
 *
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   1. against the reference itself, compiled unmodified from /root/reference
 *      into oracle/_ref/ (oracle/Makefile) and driven through
 *      oracle/ref_driver.cpp — value, every grad element, per-token lp;
 *   2. against the reference's own known-answer tests
 *      (proj/tests/test_offpolicy.cpp:55-376, acceptance.cpp:418-558) restated
 *      as pytest cases, and against committed golden fixtures
 *      (tests/golden/, generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line it follows.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "rf_oracle.h"

/* losses.cpp:83 — NaN passes through unchanged. */
static double clipd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* losses.cpp:32-39 (LossConfig::validate), codes = rf_status. */
int rfo_validate(const rfo_config* c) {
    if (!(c->clip_eps > 0.0 && c->clip_eps < 1.0)) return 1;
    if (c->eps_low < 0.0 || c->eps_high < 0.0) return 2;
    if (c->trunc_cap <= 0.0) return 3;
    if (c->kl_weight < 0.0) return 4;
    if (c->w_plus < 0.0 || c->w_minus < 0.0) return 5;
    if (c->engine_mismatch_cap < 0.0) return 6;
    if (c->variant < 0 || c->variant > 6) return 14;
    return 0;
}

/* policy.cpp:21-30 (ToyPolicy::log_probs): m = max; s = sum exp(x-m) in index
 * order; lse = m + log(s); out = x - lse. */
void rfo_log_softmax(const double* row, int32_t V, double* out) {
    double mx = row[0];
    for (int32_t v = 1; v < V; ++v)
        if (row[v] > mx) mx = row[v]; /* std::max_element: first maximal */
    double sum = 0.0;
    for (int32_t v = 0; v < V; ++v) sum += exp(row[v] - mx);
    const double lse = mx + log(sum);
    for (int32_t v = 0; v < V; ++v) out[v] = row[v] - lse;
}

/* losses.cpp:41-60 (grpo_advantages): sequential mean, population variance,
 * sd < 1e-8 -> zeros + degenerate; G < 2 -> error 13. */
int rfo_grpo_advantages(const double* rewards, const int64_t* group_offsets, int64_t num_groups,
                        double* adv, uint8_t* degenerate) {
    for (int64_t g = 0; g < num_groups; ++g) {
        const int64_t b = group_offsets[g], e = group_offsets[g + 1];
        if (e - b < 2) return 13;
    }
    for (int64_t g = 0; g < num_groups; ++g) {
        const int64_t b = group_offsets[g], e = group_offsets[g + 1];
        const double n = (double)(e - b);
        double mean = 0.0;
        for (int64_t i = b; i < e; ++i) mean += rewards[i];
        mean /= n;
        double var = 0.0;
        for (int64_t i = b; i < e; ++i) {
            const double d = rewards[i] - mean;
            var += d * d;
        }
        var /= n;
        const double sd = sqrt(var);
        if (sd < 1e-8) {
            degenerate[g] = 1;
            for (int64_t i = b; i < e; ++i) adv[i] = 0.0;
        } else {
            degenerate[g] = 0;
            for (int64_t i = b; i < e; ++i) adv[i] = (rewards[i] - mean) / sd;
        }
    }
    return 0;
}

/* The variant table shared by both aggregations.  token_mean: losses.cpp:269-319;
 * sequence_product: losses.cpp:218-251 (same formulas on trajectory scalars).
 *   r       = exp(log_ratio)   (theta / behaviour); r_sg = r (sg_anchor == policy)
 *   po      = prox / behaviour  (decoupled_ppo: exp(lq - b) per token,
 *                                exp(LR - LPX) per sequence; losses.cpp:284,224)
 *   tp      = theta / prox      (exp(lp - lq) per token, exp(LPX) per sequence)
 *   logp    = lp (token) or logp_sum (sequence) */
static void variant_math(const rfo_config* c, double r, double r_sg, double A, double po, double tp,
                         double logp, double* value, double* gw, uint8_t* flags) {
    switch (c->variant) {
        case 0: /* ppo */
        case 5: /* grpo */ {
            const double clipped = clipd(r, 1.0 - c->clip_eps, 1.0 + c->clip_eps);
            const double v1 = r * A, v2 = clipped * A;
            *value = (v2 < v1) ? v2 : v1; /* std::min(v1, v2) */
            *gw = v1 <= v2 ? r * A : (r == clipped ? r * A : 0.0);
            if (!(v1 <= v2) && r != clipped) *flags |= 0x01;
            break;
        }
        case 1: /* decoupled_ppo */ {
            const double clipped = clipd(tp, 1.0 - c->clip_eps, 1.0 + c->clip_eps);
            const double v1 = r * A, v2 = po * clipped * A;
            *value = (v2 < v1) ? v2 : v1;
            *gw = v1 <= v2 ? r * A : (tp == clipped ? po * tp * A : 0.0);
            if (!(v1 <= v2) && tp != clipped) *flags |= 0x01;
            break;
        }
        case 2: /* tis */ {
            const double w = clipd(r_sg, 0.0, c->trunc_cap);
            *value = w * A * logp;
            *gw = w * A;
            if (r_sg < 0.0 || r_sg > c->trunc_cap) *flags |= 0x01;
            break;
        }
        case 6: /* naive_is */
            *value = r_sg * A * logp;
            *gw = r_sg * A;
            break;
        case 3: /* cispo */ {
            const double lo = 1.0 - c->eps_low, hi = 1.0 + c->eps_high;
            const double w = clipd(r_sg, lo, hi);
            *value = w * A * logp;
            *gw = w * A;
            if (r_sg < lo || r_sg > hi) *flags |= 0x01;
            break;
        }
        case 4: /* topr */ {
            double w;
            if (A > 0.0) {
                w = c->w_plus;
                *flags |= 0x02;
            } else {
                w = c->w_minus * clipd(r_sg, 0.0, c->trunc_cap);
                if (r_sg < 0.0 || r_sg > c->trunc_cap) *flags |= 0x01;
            }
            *value = w * A * logp;
            *gw = w * A;
            break;
        }
        default:
            *value = 0.0;
            *gw = 0.0;
    }
}

/* KL(pi || ref) at one row and the KL gradient coefficient rows
 * (kl_and_grad, losses.cpp:118-133). */
static double row_kl(const double* lp, const double* lq, int32_t V) {
    double kl = 0.0;
    for (int32_t v = 0; v < V; ++v) kl += exp(lp[v]) * (lp[v] - lq[v]);
    return kl;
}

/* loss_and_grad (losses.cpp:137-331) on the packed layout.
 * Trajectory i = tokens [seq_offsets[i], seq_offsets[i+1]); every token t reads
 * row (row_of_token ? row_of_token[t] : t).  Per-token dlogits rows are
 *   k_t * (onehot(tok_t) - p_row)            (LogProbGrad::add/flush, losses.cpp:87-115)
 * plus, for grpo with kl_weight > 0, the KL term of kl_and_grad per token.
 * Summing dlogits rows per shared row reproduces the reference's [C x V] grad. */
int rfo_loss_and_grad(const rfo_config* c, const rfo_batch* b, rfo_outputs* o) {
    int st = rfo_validate(c);
    if (st) return st;
    if (b->num_seqs <= 0 || b->num_tokens <= 0) return 7;
    const int needs_prox = c->variant == 1;
    const int needs_ref = c->variant == 5 && c->kl_weight > 0.0;
    if (needs_prox && !b->prox_logp) return 8;
    if (needs_ref && !b->ref_logits) return 9;
    if (c->engine_mismatch_cap > 0.0 && !b->engine_logp) return 11;
    for (int64_t i = 0; i < b->num_seqs; ++i)
        if (b->seq_offsets[i + 1] <= b->seq_offsets[i]) return 10;

    const int32_t V = b->vocab;
    double* lp_row = (double*)malloc(sizeof(double) * (size_t)V);
    double* lq_row = needs_ref ? (double*)malloc(sizeof(double) * (size_t)V) : NULL;
    const int64_t t_base = b->seq_offsets[0];
    const double inv_n = 1.0 / (double)b->global_num_seqs;
    const double inv_t = 1.0 / (double)b->global_num_tokens;
    double value_total = 0.0;
    int err = 0;

    for (int64_t i = 0; i < b->num_seqs && !err; ++i) {
        const int64_t t0 = b->seq_offsets[i] - t_base, t1 = b->seq_offsets[i + 1] - t_base;
        const int64_t len = t1 - t0;
        const double A = b->advantages[i];
        const double seq_scale = b->normalization == 0 ? inv_n : inv_t * (double)len;
        const double token_scale = b->normalization == 0 ? inv_n / (double)len : inv_t;

        if (c->aggregation == 1) {
            /* sequence_product: losses.cpp:180-259. */
            double log_ratio = 0.0, logp_sum = 0.0, log_prox_ratio = 0.0, log_mismatch = 0.0;
            for (int64_t t = t0; t < t1; ++t) {
                const int64_t row = b->row_of_token ? b->row_of_token[t] : t;
                rfo_log_softmax(b->logits + row * b->row_stride, V, lp_row);
                const double lp = lp_row[b->token_ids[t]];
                if (o->token_logp) o->token_logp[t] = lp;
                if (o->token_ratio) o->token_ratio[t] = exp(lp - b->behavior_logp[t]);
                log_ratio += lp - b->behavior_logp[t];
                logp_sum += lp;
                if (needs_prox) log_prox_ratio += lp - b->prox_logp[t];
                if (c->engine_mismatch_cap > 0.0) log_mismatch += b->behavior_logp[t] - b->engine_logp[t];
            }
            const double em = exp(log_mismatch);
            const double m = c->engine_mismatch_cap > 0.0
                                 ? ((c->engine_mismatch_cap < em) ? c->engine_mismatch_cap : em)
                                 : 1.0; /* losses.cpp:207-209 */
            const double r = exp(log_ratio);
            uint8_t flags = 0;
            if (c->engine_mismatch_cap > 0.0 && em > c->engine_mismatch_cap) flags |= 0x04;
            if (!isfinite(r)) {
                flags |= 0x08;
                err = 12;
            }
            double value = 0.0, gw = 0.0;
            const double po = needs_prox ? exp(log_ratio - log_prox_ratio) : 0.0; /* losses.cpp:224 */
            const double tp = needs_prox ? exp(log_prox_ratio) : 0.0;             /* losses.cpp:225 */
            variant_math(c, r, r, A, po, tp, logp_sum, &value, &gw, &flags);
            const double k = b->grad_sign * seq_scale * m * gw;
            if (k == 0.0) flags |= 0x10;
            value_total += seq_scale * m * value;
            for (int64_t t = t0; t < t1; ++t) {
                const int64_t row = b->row_of_token ? b->row_of_token[t] : t;
                double tl = t == t0 ? seq_scale * m * value : 0.0;
                double kl = 0.0;
                if (needs_ref) {
                    rfo_log_softmax(b->logits + row * b->row_stride, V, lp_row);
                    rfo_log_softmax(b->ref_logits + row * b->ref_row_stride, V, lq_row);
                    kl = row_kl(lp_row, lq_row, V);
                    /* once per trajectory at 1/N == per token at 1/(N*L) for shared rows */
                    const double ks = b->normalization == 0 ? inv_n / (double)len : inv_t;
                    tl -= ks * c->kl_weight * kl;
                    value_total -= ks * c->kl_weight * kl;
                }
                if (o->token_loss) o->token_loss[t] = tl;
                if (o->token_coef) o->token_coef[t] = k;
                if (o->token_flags) o->token_flags[t] = flags;
                if (o->dlogits) {
                    if (!needs_ref) rfo_log_softmax(b->logits + row * b->row_stride, V, lp_row);
                    double* d = o->dlogits + (t)*o->dlogits_row_stride;
                    const int32_t tok = b->token_ids[t];
                    const double ks = b->normalization == 0 ? inv_n / (double)len : inv_t;
                    const double kcoef = -b->grad_sign * ks * c->kl_weight;
                    for (int32_t v = 0; v < V; ++v) {
                        const double p = exp(lp_row[v]);
                        double g = 0.0; /* LogProbGrad: grad[tok] += k; grad[v] -= k*p[v] */
                        if (k != 0.0) g = (v == tok) ? (k - k * p) : -(k * p);
                        if (needs_ref) g += kcoef * p * ((lp_row[v] - lq_row[v]) - kl);
                        d[v] = g;
                    }
                }
            }
            continue;
        }

        /* token_mean: losses.cpp:262-327. */
        for (int64_t t = t0; t < t1; ++t) {
            const int64_t row = b->row_of_token ? b->row_of_token[t] : t;
            const double* x = b->logits + row * b->row_stride;
            rfo_log_softmax(x, V, lp_row);
            const int32_t tok = b->token_ids[t];
            const double lp = lp_row[tok];
            const double bl = b->behavior_logp[t];
            const double lr = lp - bl;
            const double r = exp(lr);
            uint8_t flags = 0;
            if (!isfinite(r)) {
                flags |= 0x08;
                err = 12; /* losses.cpp:267 throws */
            }
            double m = 1.0;
            if (c->engine_mismatch_cap > 0.0) { /* losses.cpp:170-176 */
                const double em = exp(bl - b->engine_logp[t]);
                m = (c->engine_mismatch_cap < em) ? c->engine_mismatch_cap : em; /* std::min */
                if (em > c->engine_mismatch_cap) flags |= 0x04;
            }
            double value = 0.0, gw = 0.0;
            double po = 0.0, tp = 0.0;
            if (needs_prox) { /* losses.cpp:283-285 */
                const double lq = b->prox_logp[t];
                po = exp(lq - bl);
                tp = exp(lp - lq);
            }
            variant_math(c, r, r, A, po, tp, lp, &value, &gw, &flags);
            const double k = b->grad_sign * token_scale * m * gw;
            if (k == 0.0) flags |= 0x10;
            double tl = token_scale * m * value;
            value_total += token_scale * m * value;
            double kl = 0.0;
            if (needs_ref) {
                rfo_log_softmax(b->ref_logits + row * b->ref_row_stride, V, lq_row);
                kl = row_kl(lp_row, lq_row, V);
                tl -= token_scale * c->kl_weight * kl;
                value_total -= token_scale * c->kl_weight * kl;
            }
            if (o->token_logp) o->token_logp[t] = lp;
            if (o->token_ratio) o->token_ratio[t] = r;
            if (o->token_coef) o->token_coef[t] = k;
            if (o->token_loss) o->token_loss[t] = tl;
            if (o->token_flags) o->token_flags[t] = flags;
            if (o->dlogits) {
                double* d = o->dlogits + t * o->dlogits_row_stride;
                const double kcoef = -b->grad_sign * token_scale * c->kl_weight;
                for (int32_t v = 0; v < V; ++v) {
                    const double p = exp(lp_row[v]);
                    /* LogProbGrad: grad[tok] += k; grad[v] -= k * p[v]; rows with
                     * k == 0 are skipped entirely (stay +0.0). */
                    double g = 0.0;
                    if (k != 0.0) g = (v == tok) ? (k - k * p) : -(k * p);
                    if (needs_ref) g += kcoef * p * ((lp_row[v] - lq_row[v]) - kl);
                    d[v] = g;
                }
            }
        }
    }
    free(lp_row);
    free(lq_row);
    if (o->value) *o->value = value_total;
    return err;
}
