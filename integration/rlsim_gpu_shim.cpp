// rlsim_gpu_shim.cpp — the reference-side binding: rlsim's loss API
// (proj/include/rlsim/losses.hpp) implemented over the C ABI of
// include/rf_offpolicy.h, so the reference's own callers (toy_train_loop,
// bandit.cpp:41-119; experiment offpolicy mode) link unchanged against the GPU
// path.  Built by integration/Makefile together with the reference's UNMODIFIED
// bandit.cpp / policy.cpp / rng.cpp / engine.cpp (compiled from /root/reference,
// nothing copied) in place of losses.cpp.
//
// Mapping: every Trajectory = one CSR sequence whose tokens read its context
// row ("mapping B"); the ToyPolicy table goes to the GPU as f32 rows; the
// reference's seq-then-batch normalisation 1/(N*L_i) (losses.cpp:152,167);
// LossResult.grad = per-context sum of the per-token f32 dlogits rows.  The
// proximal policy's per-token log-probs come from a stats-only GPU pass over
// the prox table.  Not supported: LossInputs::sg_anchor != policy (the
// finite-difference oracle's stop-gradient pin) — reported as invalid_argument.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "rf_offpolicy.h"
#include "rlsim/losses.hpp"

namespace rlsim {

namespace {

[[noreturn]] void raise(rf_status s) { throw std::invalid_argument(rf_status_string(s)); }

rf_loss_config to_c(const LossConfig& c) {
    rf_loss_config r;
    r.variant = static_cast<int32_t>(c.variant);
    r.aggregation = static_cast<int32_t>(c.aggregation);
    r.clip_eps = c.clip_eps;
    r.eps_low = c.eps_low;
    r.eps_high = c.eps_high;
    r.trunc_cap = c.trunc_cap;
    r.kl_weight = c.kl_weight;
    r.w_plus = c.w_plus;
    r.w_minus = c.w_minus;
    r.engine_mismatch_cap = c.engine_mismatch_cap;
    return r;
}

std::vector<float> table_f32(const ToyPolicy& p) {
    std::vector<float> t(p.logits().size());
    for (size_t i = 0; i < t.size(); ++i) t[i] = static_cast<float>(p.logits()[i]);
    return t;
}

int device_id() {
    const char* e = std::getenv("RF_DEVICE");
    return e ? std::atoi(e) : 0;
}

}  // namespace

const char* to_string(LossVariant v) noexcept { return rf_loss_variant_name(static_cast<int32_t>(v)); }

LossVariant loss_variant_from_string(const std::string& s) {
    int32_t v = 0;
    if (rf_loss_variant_from_name(s.c_str(), &v) != RF_OK) throw std::invalid_argument("unknown loss variant: " + s);
    return static_cast<LossVariant>(v);
}

void LossConfig::validate() const {
    const rf_loss_config c = to_c(*this);
    const rf_status s = rf_loss_config_validate(&c);
    if (s != RF_OK) raise(s);
}

GroupAdvantages grpo_advantages(const std::vector<double>& rewards) {
    // One group on the host-side mirror would need a device round trip per group;
    // the reference callers pass one group at a time, so batch-of-one K1 launch.
    if (rewards.size() < 2) raise(RF_ERR_GROUP_TOO_SMALL);
    GroupAdvantages out;
    out.values.resize(rewards.size());
    // K1 through the device API on a tiny buffer (the ABI has no host-buffer K1).
    const int64_t n = static_cast<int64_t>(rewards.size());
    cudaSetDevice(device_id());
    double *d_r = nullptr, *d_a = nullptr;
    int64_t* d_go = nullptr;
    uint8_t* d_deg = nullptr;
    int32_t* d_st = nullptr;
    cudaMalloc(&d_r, n * 8);
    cudaMalloc(&d_a, n * 8);
    cudaMalloc(&d_go, 16);
    cudaMalloc(&d_deg, 1);
    cudaMalloc(&d_st, 4);
    const int64_t go[2] = {0, n};
    cudaMemcpy(d_r, rewards.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_go, go, 16, cudaMemcpyHostToDevice);
    rf_batch b{};
    b.num_groups = 1;
    b.num_seqs = n;
    b.rewards = d_r;
    b.group_offsets = d_go;
    rf_outputs o{};
    o.advantages_out = d_a;
    o.group_degenerate = d_deg;
    o.device_status = d_st;
    const rf_status s = rf_grpo_advantages(&b, &o, nullptr);
    uint8_t deg = 0;
    cudaMemcpy(out.values.data(), d_a, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&deg, d_deg, 1, cudaMemcpyDeviceToHost);
    for (void* p : {static_cast<void*>(d_r), static_cast<void*>(d_a), static_cast<void*>(d_go),
                    static_cast<void*>(d_deg), static_cast<void*>(d_st)})
        cudaFree(p);
    if (s != RF_OK) raise(s);
    out.degenerate = deg != 0;
    return out;
}

TrajectoryRatio trajectory_ratio(const ToyPolicy& policy, const Trajectory& traj) {
    // per-token exp(lp - b) from the GPU stats pass (losses.cpp:62-79 semantics)
    if (traj.tokens.empty()) throw std::invalid_argument("trajectory_ratio: empty trajectory");
    if (traj.behavior_logp.size() != traj.tokens.size())
        throw std::invalid_argument("trajectory_ratio: behavior log-probs missing");
    Trajectory t = traj;
    t.advantage = 0.0;
    LossConfig cfg;
    cfg.variant = LossVariant::naive_is;
    const std::vector<float> tab = table_f32(policy);
    const int64_t T = static_cast<int64_t>(t.tokens.size());
    std::vector<int32_t> tok(t.tokens.begin(), t.tokens.end()), rows(T, t.context), sot(T, 0);
    std::vector<int64_t> offs = {0, T};
    std::vector<double> adv = {0.0}, ratio(T), scal(RF_NUM_SCALARS);
    rf_loss_config c = to_c(cfg);
    rf_batch b{};
    b.num_tokens = T;
    b.num_seqs = 1;
    b.vocab = policy.vocab();
    b.logits_dtype = RF_DTYPE_F32;
    b.logits = tab.data();
    b.logits_row_stride = policy.vocab();
    b.row_of_token = rows.data();
    b.token_ids = tok.data();
    b.seq_of_token = sot.data();
    b.seq_offsets = offs.data();
    b.advantages = adv.data();
    b.logp_dtype = RF_DTYPE_F64;
    b.behavior_logp = t.behavior_logp.data();
    b.global_num_seqs = 1;
    b.global_num_tokens = T;
    b.grad_sign = 1.0;
    rf_outputs o{};
    o.token_ratio = ratio.data();
    o.scalars = scal.data();
    int32_t st = 0;
    o.device_status = &st;
    const rf_status s = rf_loss_and_grad_host(&c, &b, &o, device_id(), 0);
    if (s == RF_ERR_NONFINITE_RATIO) throw std::invalid_argument("trajectory_ratio: non-finite log ratio");
    if (s != RF_OK) raise(s);
    TrajectoryRatio r;
    double log_sum = 0.0;
    for (int64_t i = 0; i < T; ++i) {
        r.per_token.push_back(ratio[static_cast<size_t>(i)]);
        log_sum += std::log(ratio[static_cast<size_t>(i)]);
    }
    r.product = std::exp(log_sum);
    return r;
}

LossResult loss_and_grad(const LossConfig& config, const ToyPolicy& policy, const std::vector<Trajectory>& batch,
                         const LossInputs& aux) {
    config.validate();
    if (batch.empty()) raise(RF_ERR_EMPTY_BATCH);
    const bool needs_prox = config.variant == LossVariant::decoupled_ppo;
    const bool needs_ref = config.variant == LossVariant::grpo && config.kl_weight > 0.0;
    if (needs_prox && aux.prox == nullptr) raise(RF_ERR_MISSING_PROX);
    if (needs_ref && aux.ref == nullptr) raise(RF_ERR_MISSING_REF);
    if (aux.sg_anchor != nullptr && aux.sg_anchor != &policy)
        throw std::invalid_argument("loss_and_grad: sg_anchor other than the policy is not supported on the GPU path");
    const int C = policy.contexts(), V = policy.vocab();
    // packed batch (mapping B)
    std::vector<int32_t> tok, rows, sot;
    std::vector<int64_t> offs = {0};
    std::vector<double> adv, beh, eng;
    const bool cap = config.engine_mismatch_cap > 0.0;
    for (size_t i = 0; i < batch.size(); ++i) {
        const Trajectory& t = batch[i];
        if (t.tokens.empty()) raise(RF_ERR_EMPTY_TRAJECTORY);
        if (cap && t.engine_logp.size() != t.tokens.size()) raise(RF_ERR_MISSING_ENGINE_LOGP);
        for (size_t k = 0; k < t.tokens.size(); ++k) {
            tok.push_back(t.tokens[k]);
            rows.push_back(t.context);
            sot.push_back(static_cast<int32_t>(i));
            beh.push_back(t.behavior_logp.at(k));
            if (cap) eng.push_back(t.engine_logp[k]);
        }
        offs.push_back(static_cast<int64_t>(tok.size()));
        adv.push_back(t.advantage);
    }
    const int64_t T = static_cast<int64_t>(tok.size()), N = static_cast<int64_t>(batch.size());
    const std::vector<float> tab = table_f32(policy);
    rf_batch b{};
    b.num_tokens = T;
    b.num_seqs = N;
    b.vocab = V;
    b.logits_dtype = RF_DTYPE_F32;
    b.logits = tab.data();
    b.logits_row_stride = V;
    b.row_of_token = rows.data();
    b.token_ids = tok.data();
    b.seq_of_token = sot.data();
    b.seq_offsets = offs.data();
    b.advantages = adv.data();
    b.logp_dtype = RF_DTYPE_F64;
    b.normalization = RF_NORM_SEQ_THEN_BATCH;
    b.behavior_logp = beh.data();
    b.engine_logp = cap ? eng.data() : nullptr;
    b.global_num_seqs = N;
    b.global_num_tokens = T;
    b.grad_sign = 1.0;
    std::vector<double> scal(RF_NUM_SCALARS);
    int32_t st = 0;
    std::vector<double> lq;
    std::vector<float> prox_tab, ref_tab;
    if (needs_prox) {  // per-token log pi_prox(token): stats-only GPU pass over the prox table
        prox_tab = table_f32(*aux.prox);
        rf_batch q = b;
        q.logits = prox_tab.data();
        q.engine_logp = nullptr;
        rf_loss_config qc = to_c(LossConfig{});
        qc.variant = RF_NAIVE_IS;
        lq.resize(static_cast<size_t>(T));
        rf_outputs qo{};
        qo.token_logp = lq.data();
        qo.scalars = scal.data();
        qo.device_status = &st;
        const rf_status s = rf_loss_and_grad_host(&qc, &q, &qo, device_id(), 0);
        if (s != RF_OK && s != RF_ERR_NONFINITE_RATIO) raise(s);
        b.prox_logp = lq.data();
    }
    if (needs_ref) {
        ref_tab = table_f32(*aux.ref);
        b.ref_logits = ref_tab.data();
        b.ref_row_stride = V;
    }
    std::vector<float> dl(static_cast<size_t>(T) * V);
    rf_outputs o{};
    o.dlogits = dl.data();
    o.dlogits_dtype = RF_DTYPE_F32;
    o.dlogits_row_stride = V;
    std::fill(scal.begin(), scal.end(), 0.0);
    o.scalars = scal.data();
    o.device_status = &st;
    rf_loss_config c = to_c(config);
    const rf_status s = rf_loss_and_grad_host(&c, &b, &o, device_id(), 0);
    if (s != RF_OK) raise(s);
    LossResult res;
    res.value = scal[RF_SCALAR_LOSS];
    res.grad.assign(static_cast<size_t>(C) * V, 0.0);
    for (int64_t t = 0; t < T; ++t) {  // LogProbGrad's per-context accumulation (losses.cpp:95-108)
        const float* d = dl.data() + static_cast<size_t>(t) * V;
        double* g = res.grad.data() + static_cast<size_t>(rows[static_cast<size_t>(t)]) * V;
        for (int v = 0; v < V; ++v) g[v] += static_cast<double>(d[v]);
    }
    return res;
}

}  // namespace rlsim
