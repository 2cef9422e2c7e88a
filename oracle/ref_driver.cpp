// ref_driver.cpp — TEST / BASELINE INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver around the UNMODIFIED reference library (rlsim),
// compiled together with the reference's own sources from /root/reference by
// oracle/Makefile into oracle/_ref/librlsim_ref.so.  It marshals flat arrays
// into rlsim::ToyPolicy / rlsim::Trajectory (policy.hpp:12-51) and calls the
// reference entry points:
//   rlsim::grpo_advantages      losses.cpp:41-60
//   rlsim::loss_and_grad        losses.cpp:137-331
//   rlsim::ToyPolicy::log_probs policy.cpp:21-30
//   rlsim::toy_train_loop       bandit.cpp:41-119
// Used (a) by tests/ to pin oracle/rf_oracle.c and to generate golden fixtures,
// (b) by bench.py --impl reference / cpu_baseline to time the reference's own
// CPU implementation on host cores.  Nothing here is product code.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "rlsim/bandit.hpp"
#include "rlsim/gradcheck.hpp"
#include "rlsim/losses.hpp"
#include "rlsim/policy.hpp"

using namespace rlsim;

namespace {

void set_err(char* buf, int len, const char* msg) {
    if (buf && len > 0) {
        std::strncpy(buf, msg, static_cast<size_t>(len) - 1);
        buf[len - 1] = '\0';
    }
}

LossConfig make_config(int32_t variant, int32_t aggregation, const double* p) {
    LossConfig c;
    c.variant = static_cast<LossVariant>(variant);
    c.aggregation = static_cast<RatioAggregation>(aggregation);
    c.clip_eps = p[0];
    c.eps_low = p[1];
    c.eps_high = p[2];
    c.trunc_cap = p[3];
    c.kl_weight = p[4];
    c.w_plus = p[5];
    c.w_minus = p[6];
    c.engine_mismatch_cap = p[7];
    return c;
}

std::vector<Trajectory> make_batch(int64_t num_traj, const int32_t* traj_context, const int64_t* traj_offsets,
                                   const int32_t* tokens, const double* advantages, const double* behavior_logp,
                                   const double* engine_logp) {
    std::vector<Trajectory> batch(static_cast<size_t>(num_traj));
    for (int64_t i = 0; i < num_traj; ++i) {
        Trajectory& t = batch[static_cast<size_t>(i)];
        t.context = traj_context[i];
        t.advantage = advantages[i];
        for (int64_t k = traj_offsets[i]; k < traj_offsets[i + 1]; ++k) {
            t.tokens.push_back(tokens[k]);
            t.behavior_logp.push_back(behavior_logp[k]);
            if (engine_logp) t.engine_logp.push_back(engine_logp[k]);
        }
    }
    return batch;
}

}  // namespace

extern "C" {

int ref_grpo_advantages(const double* rewards, int64_t n, double* out, uint8_t* degenerate, char* err,
                        int errlen) {
    try {
        std::vector<double> r(rewards, rewards + n);
        const GroupAdvantages a = grpo_advantages(r);
        for (int64_t i = 0; i < n; ++i) out[i] = a.values[static_cast<size_t>(i)];
        *degenerate = a.degenerate ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int ref_variant_from_string(const char* name, int32_t* out, char* err, int errlen) {
    try {
        *out = static_cast<int32_t>(loss_variant_from_string(name));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

const char* ref_variant_to_string(int32_t v) { return to_string(static_cast<LossVariant>(v)); }

int ref_validate(int32_t variant, int32_t aggregation, const double* params, char* err, int errlen) {
    try {
        make_config(variant, aggregation, params).validate();
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// loss_and_grad over trajectories.  logits/prox/ref are [contexts x vocab]
// fp64 tables (prox/ref nullable).  grad_out (nullable) receives the [C x V]
// gradient.
int ref_loss_and_grad(int32_t variant, int32_t aggregation, const double* params, int32_t contexts,
                      int32_t vocab, const double* logits, const double* prox_logits, const double* ref_logits,
                      int64_t num_traj, const int32_t* traj_context, const int64_t* traj_offsets,
                      const int32_t* tokens, const double* advantages, const double* behavior_logp,
                      const double* engine_logp, double* value_out, double* grad_out, char* err, int errlen) {
    try {
        const size_t n = static_cast<size_t>(contexts) * static_cast<size_t>(vocab);
        ToyPolicy policy(contexts, vocab, std::vector<double>(logits, logits + n));
        ToyPolicy prox(contexts, vocab);
        ToyPolicy ref(contexts, vocab);
        LossInputs aux;
        if (prox_logits) {
            prox = ToyPolicy(contexts, vocab, std::vector<double>(prox_logits, prox_logits + n));
            aux.prox = &prox;
        }
        if (ref_logits) {
            ref = ToyPolicy(contexts, vocab, std::vector<double>(ref_logits, ref_logits + n));
            aux.ref = &ref;
        }
        const std::vector<Trajectory> batch =
            make_batch(num_traj, traj_context, traj_offsets, tokens, advantages, behavior_logp, engine_logp);
        const LossResult res = loss_and_grad(make_config(variant, aggregation, params), policy, batch, aux);
        *value_out = res.value;
        if (grad_out) std::memcpy(grad_out, res.grad.data(), n * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// ToyPolicy::log_probs of the given rows.
int ref_log_probs(int32_t contexts, int32_t vocab, const double* logits, int64_t count, const int32_t* rows,
                  double* out) {
    const size_t n = static_cast<size_t>(contexts) * static_cast<size_t>(vocab);
    ToyPolicy policy(contexts, vocab, std::vector<double>(logits, logits + n));
    for (int64_t i = 0; i < count; ++i) {
        const std::vector<double> lp = policy.log_probs(rows[i]);
        std::memcpy(out + i * vocab, lp.data(), sizeof(double) * static_cast<size_t>(vocab));
    }
    return 0;
}

// trajectory_ratio (losses.cpp:62-79) of one trajectory.
int ref_trajectory_ratio(int32_t contexts, int32_t vocab, const double* logits, int32_t context, int64_t len,
                         const int32_t* tokens, const double* behavior_logp, double* per_token, double* product,
                         char* err, int errlen) {
    try {
        const size_t n = static_cast<size_t>(contexts) * static_cast<size_t>(vocab);
        ToyPolicy policy(contexts, vocab, std::vector<double>(logits, logits + n));
        Trajectory t;
        t.context = context;
        t.tokens.assign(tokens, tokens + len);
        t.behavior_logp.assign(behavior_logp, behavior_logp + len);
        const TrajectoryRatio r = trajectory_ratio(policy, t);
        for (int64_t i = 0; i < len; ++i) per_token[i] = r.per_token[static_cast<size_t>(i)];
        *product = r.product;
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// finite_diff_check (gradcheck.cpp:59-96): max rel error, checked, flagged.
int ref_finite_diff(int32_t variant, int32_t aggregation, const double* params, int32_t contexts, int32_t vocab,
                    const double* logits, const double* prox_logits, const double* ref_logits, int64_t num_traj,
                    const int32_t* traj_context, const int64_t* traj_offsets, const int32_t* tokens,
                    const double* advantages, const double* behavior_logp, const double* engine_logp, double h,
                    double* max_rel_err, int64_t* checked, int64_t* flagged, char* err, int errlen) {
    try {
        const size_t n = static_cast<size_t>(contexts) * static_cast<size_t>(vocab);
        ToyPolicy policy(contexts, vocab, std::vector<double>(logits, logits + n));
        ToyPolicy prox(contexts, vocab), ref(contexts, vocab);
        LossInputs aux;
        if (prox_logits) {
            prox = ToyPolicy(contexts, vocab, std::vector<double>(prox_logits, prox_logits + n));
            aux.prox = &prox;
        }
        if (ref_logits) {
            ref = ToyPolicy(contexts, vocab, std::vector<double>(ref_logits, ref_logits + n));
            aux.ref = &ref;
        }
        const auto batch =
            make_batch(num_traj, traj_context, traj_offsets, tokens, advantages, behavior_logp, engine_logp);
        const GradReport rep = finite_diff_check(make_config(variant, aggregation, params), policy, batch, h, aux);
        *max_rel_err = rep.max_rel_error;
        *checked = static_cast<int64_t>(rep.checked);
        *flagged = static_cast<int64_t>(rep.flagged);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// A proximal-policy table whose log-softmax at (row, token) equals lq exactly
// in exact arithmetic: the token's logit is moved, every other logit is kept.
// Lets the reference (which needs a full prox ToyPolicy, LossInputs::prox)
// consume the per-token prox log-probs of the packed layout.
void ref_build_prox_table(int32_t rows, int32_t vocab, const double* logits, const int32_t* tokens,
                          const double* lq, double* out) {
    for (int32_t c = 0; c < rows; ++c) {
        const double* x = logits + static_cast<size_t>(c) * vocab;
        double* y = out + static_cast<size_t>(c) * vocab;
        std::memcpy(y, x, sizeof(double) * static_cast<size_t>(vocab));
        const int32_t tok = tokens[c];
        double mx = -INFINITY;
        for (int32_t v = 0; v < vocab; ++v)
            if (v != tok && x[v] > mx) mx = x[v];
        double s = 0.0;
        for (int32_t v = 0; v < vocab; ++v)
            if (v != tok) s += std::exp(x[v] - mx);
        y[tok] = lq[c] + mx + std::log(s) - std::log1p(-std::exp(lq[c]));
    }
}

// Time the reference loss_and_grad on mapping-A rows (one length-1 trajectory
// per token, context = its own row) with `threads` host threads, each owning a
// contiguous shard of rows and its own ToyPolicy (the reference is
// single-threaded and reentrant).  Returns wall seconds of `reps` repetitions
// of the parallel region (setup excluded); value_out = sum of shard values.
double ref_bench_mapping_a(int32_t threads, int32_t variant, const double* params, int32_t rows, int32_t vocab,
                           const double* logits, const double* prox_logits, const int32_t* tokens,
                           const double* advantages, const double* behavior_logp, const double* engine_logp,
                           int32_t reps, double* value_out) {
    if (threads < 1) threads = 1;
    if (threads > rows) threads = rows;
    struct Shard {
        ToyPolicy policy{1, 2};
        ToyPolicy prox{1, 2};
        std::vector<Trajectory> batch;
        double value = 0.0;
    };
    std::vector<Shard> shards(static_cast<size_t>(threads));
    const LossConfig cfg = make_config(variant, 0, params);
    for (int32_t s = 0; s < threads; ++s) {
        const int32_t r0 = static_cast<int32_t>(static_cast<int64_t>(rows) * s / threads);
        const int32_t r1 = static_cast<int32_t>(static_cast<int64_t>(rows) * (s + 1) / threads);
        const int32_t n = r1 - r0;
        Shard& sh = shards[static_cast<size_t>(s)];
        const size_t off = static_cast<size_t>(r0) * vocab, cnt = static_cast<size_t>(n) * vocab;
        sh.policy = ToyPolicy(n, vocab, std::vector<double>(logits + off, logits + off + cnt));
        if (prox_logits) sh.prox = ToyPolicy(n, vocab, std::vector<double>(prox_logits + off, prox_logits + off + cnt));
        for (int32_t c = 0; c < n; ++c) {
            Trajectory t;
            t.context = c;
            t.tokens = {tokens[r0 + c]};
            t.advantage = advantages[r0 + c];
            t.behavior_logp = {behavior_logp[r0 + c]};
            if (engine_logp) t.engine_logp = {engine_logp[r0 + c]};
            sh.batch.push_back(std::move(t));
        }
    }
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<std::thread> pool;
    std::chrono::steady_clock::time_point t0, t1;
    for (int32_t s = 0; s < threads; ++s) {
        pool.emplace_back([&, s] {
            Shard& sh = shards[static_cast<size_t>(s)];
            LossInputs aux;
            if (prox_logits) aux.prox = &sh.prox;
            ready.fetch_add(1);
            while (!go.load(std::memory_order_acquire)) {
            }
            for (int32_t r = 0; r < reps; ++r) sh.value = loss_and_grad(cfg, sh.policy, sh.batch, aux).value;
        });
    }
    while (ready.load() < threads) {
    }
    t0 = std::chrono::steady_clock::now();
    go.store(true, std::memory_order_release);
    for (auto& th : pool) th.join();
    t1 = std::chrono::steady_clock::now();
    double v = 0.0;
    for (const auto& sh : shards) v += sh.value;
    if (value_out) *value_out = v;
    return std::chrono::duration<double>(t1 - t0).count();
}

// toy_train_loop (bandit.cpp:41-119).  curve arrays sized `steps`.
int ref_train_loop(int32_t contexts, int32_t arms, int32_t group_size, int32_t traj_len, int32_t steps, double lr,
                   double reward_noise, int64_t async_lag, uint64_t seed, int32_t variant, int32_t aggregation,
                   const double* params, double* final_reward, double* grad_norm_variance, double* curve_reward,
                   double* curve_gnorm, int64_t* curve_staleness, char* err, int errlen) {
    try {
        TrainLoopConfig cfg;
        cfg.contexts = contexts;
        cfg.arms = arms;
        cfg.group_size = group_size;
        cfg.traj_len = traj_len;
        cfg.steps = steps;
        cfg.lr = lr;
        cfg.reward_noise = reward_noise;
        cfg.async_lag = async_lag;
        cfg.seed = seed;
        cfg.loss = make_config(variant, aggregation, params);
        const TrainLoopResult res = toy_train_loop(cfg);
        *final_reward = res.final_reward;
        *grad_norm_variance = res.grad_norm_variance;
        for (size_t i = 0; i < res.curve.size(); ++i) {
            curve_reward[i] = res.curve[i].expected_reward;
            curve_gnorm[i] = res.curve[i].grad_norm;
            curve_staleness[i] = res.curve[i].staleness;
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// RngStream draws (rng.hpp:44-84) for cross-checking the synthetic-input
// generator: kind 0 = uniform01, 1 = normal, 2 = next_u64 (as double bits).
void ref_rng_draws(uint64_t seed, const char* name, int32_t kind, int64_t n, double* out) {
    RngStream rng(seed, std::string_view(name));
    for (int64_t i = 0; i < n; ++i) {
        if (kind == 0) out[i] = rng.uniform01();
        else if (kind == 1) out[i] = rng.normal();
        else {
            const uint64_t u = rng.next_u64();
            std::memcpy(&out[i], &u, sizeof(u));
        }
    }
}

}  // extern "C"
