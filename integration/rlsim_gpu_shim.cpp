// rlsim_gpu_shim.cpp — the reference-side binding: rlsim's loss API
// (proj/include/rlsim/losses.hpp) implemented over the C ABI of
// include/rf_offpolicy.h, so the reference's own callers (toy_train_loop,
// bandit.cpp:41-119; the experiment `offpolicy` mode, experiment.cpp:589-622)
// link unchanged against the GPU path.  Built by integration/Makefile together
// with the reference's UNMODIFIED sources (compiled from /root/reference, nothing
// copied) in place of losses.cpp.
//
// Mapping: every Trajectory = one CSR sequence whose tokens read its context
// row ("mapping B"); the ToyPolicy table goes to the GPU as f32 rows; the
// reference's seq-then-batch normalisation 1/(N*L_i) (losses.cpp:152,167).  Per
// call: one upload of the table(s) and the packed batch, the proximal policy's
// per-token log-probs from a stats-only pass over the prox table (device to
// device), the fused loss + f32 dlogits, then LossResult.grad = the per-context
// fp64 sum of the dlogits rows on the device (rf_rows_segment_sum), and one
// download of grad + scalars + status.  Device buffers live in a per-thread
// context and only grow.  Not supported: LossInputs::sg_anchor != policy (the
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

void cuda_ok(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

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

int device_id() {
    const char* e = std::getenv("RF_DEVICE");
    return e ? std::atoi(e) : 0;
}

// A grow-only device buffer.
struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <typename T>
    T* get(size_t n) {
        const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cuda_ok(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return static_cast<T*>(p);
    }
    template <typename T>
    T* put(const T* src, size_t n, cudaStream_t s) {
        T* d = get<T>(n);
        if (n) cuda_ok(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
        return d;
    }
};

// Per-thread device context: stream + buffers reused across calls.
struct Ctx {
    int dev = -1;
    cudaStream_t s = nullptr;
    DBuf table, prox, ref, tok, rows, sot, offs, adv, beh, eng, lq, lp, ratio, dl, grad, segoffs, segrows, scal, st,
        ws, rew, gofs, deg;
    Ctx() {
        dev = device_id();
        cuda_ok(cudaSetDevice(dev));
        cuda_ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
};

Ctx& ctx() {
    thread_local Ctx c;
    cuda_ok(cudaSetDevice(c.dev));
    return c;
}

float* upload_table(DBuf& buf, const ToyPolicy& p, cudaStream_t s) {
    std::vector<float> t(p.logits().size());
    for (size_t i = 0; i < t.size(); ++i) t[i] = static_cast<float>(p.logits()[i]);
    float* d = buf.get<float>(t.size());
    cuda_ok(cudaMemcpyAsync(d, t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    cuda_ok(cudaStreamSynchronize(s));  // t is a stack buffer
    return d;
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
    // The reference's callers pass one group per call (bandit.cpp:76): one K1 launch on
    // the context's persistent buffers, one round trip.
    if (rewards.size() < 2) raise(RF_ERR_GROUP_TOO_SMALL);  // losses.cpp:42
    Ctx& c = ctx();
    const int64_t n = static_cast<int64_t>(rewards.size());
    const int64_t go[2] = {0, n};
    rf_batch b{};
    b.num_groups = 1;
    b.num_seqs = n;
    b.rewards = c.rew.put(rewards.data(), rewards.size(), c.s);
    b.group_offsets = c.gofs.put(go, 2, c.s);
    rf_outputs o{};
    o.advantages_out = c.adv.get<double>(static_cast<size_t>(n));
    o.group_degenerate = c.deg.get<uint8_t>(1);
    o.device_status = c.st.get<int32_t>(1);
    cuda_ok(cudaMemsetAsync(o.device_status, 0, 4, c.s));
    const rf_status s = rf_grpo_advantages(&b, &o, c.s);
    if (s != RF_OK) raise(s);
    GroupAdvantages out;
    out.values.resize(rewards.size());
    uint8_t deg = 0;
    cuda_ok(cudaMemcpyAsync(out.values.data(), o.advantages_out, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost,
                            c.s));
    cuda_ok(cudaMemcpyAsync(&deg, o.group_degenerate, 1, cudaMemcpyDeviceToHost, c.s));
    cuda_ok(cudaStreamSynchronize(c.s));
    out.degenerate = deg != 0;
    return out;
}

namespace {

// The packed batch (mapping B) on the device: one CSR sequence per trajectory, every
// token reading its context row.  Host-side validation of what the reference leaves
// as UB (token / context ranges).
struct Packed {
    std::vector<int32_t> tok, rows, sot;
    std::vector<int64_t> offs{0};
    std::vector<double> adv, beh, eng;
};

void fill_batch(rf_batch& b, Ctx& c, const Packed& pk, const float* table, int V, bool with_eng) {
    const size_t T = pk.tok.size(), N = pk.adv.size();
    b.num_tokens = static_cast<int64_t>(T);
    b.num_seqs = static_cast<int64_t>(N);
    b.vocab = V;
    b.logits_dtype = RF_DTYPE_F32;
    b.logits = table;
    b.logits_row_stride = V;
    b.row_of_token = c.rows.put(pk.rows.data(), T, c.s);
    b.token_ids = c.tok.put(pk.tok.data(), T, c.s);
    b.seq_of_token = c.sot.put(pk.sot.data(), T, c.s);
    b.seq_offsets = c.offs.put(pk.offs.data(), N + 1, c.s);
    b.advantages = c.adv.put(pk.adv.data(), N, c.s);
    b.logp_dtype = RF_DTYPE_F64;
    b.normalization = RF_NORM_SEQ_THEN_BATCH;
    b.behavior_logp = c.beh.put(pk.beh.data(), T, c.s);
    b.engine_logp = with_eng ? c.eng.put(pk.eng.data(), T, c.s) : nullptr;
    b.global_num_seqs = static_cast<int64_t>(N);
    b.global_num_tokens = static_cast<int64_t>(T);
    b.grad_sign = 1.0;
}

void attach_common(rf_outputs& o, Ctx& c, const rf_loss_config& cfg, const rf_batch& b) {
    o.scalars = c.scal.get<double>(RF_NUM_SCALARS);
    o.device_status = c.st.get<int32_t>(1);
    const size_t wsb = rf_workspace_bytes(&cfg, &b);
    o.workspace = c.ws.get<uint8_t>(wsb);
    o.workspace_bytes = std::max<size_t>(wsb, 16);
    const rf_status z = rf_zero_scalars(&o, c.s);
    if (z != RF_OK) raise(z);
}

// Per-token log pi(token) of `table` over the batch (stats-only pass: no dlogits,
// the device status of the ratio against `beh` is ignored).
double* token_logp(Ctx& c, DBuf& out, const rf_batch& b0) {
    rf_batch q = b0;
    q.engine_logp = nullptr;
    q.prox_logp = nullptr;
    q.ref_logits = nullptr;
    rf_loss_config qc;
    rf_loss_config_default(&qc);
    qc.variant = RF_NAIVE_IS;
    rf_outputs o{};
    o.token_logp = out.get<double>(static_cast<size_t>(b0.num_tokens));
    attach_common(o, c, qc, q);
    const rf_status s = rf_loss_and_grad(&qc, &q, &o, c.s);
    if (s != RF_OK) raise(s);
    return o.token_logp;
}

}  // namespace

TrajectoryRatio trajectory_ratio(const ToyPolicy& policy, const Trajectory& traj) {
    // losses.cpp:62-79: lp from the GPU log-softmax, the log ratio and its product
    // exactly as the reference forms them (the same throw sites).
    if (traj.tokens.empty()) throw std::invalid_argument("trajectory_ratio: empty trajectory");
    if (traj.behavior_logp.size() != traj.tokens.size())
        throw std::invalid_argument("trajectory_ratio: behavior log-probs missing");
    Ctx& c = ctx();
    const int V = policy.vocab();
    Packed pk;
    for (size_t k = 0; k < traj.tokens.size(); ++k) {
        if (traj.tokens[k] < 0 || traj.tokens[k] >= V) raise(RF_ERR_TOKEN_OUT_OF_RANGE);
        pk.tok.push_back(traj.tokens[k]);
        pk.rows.push_back(traj.context);
        pk.sot.push_back(0);
        pk.beh.push_back(traj.behavior_logp[k]);
    }
    if (traj.context < 0 || traj.context >= policy.contexts()) raise(RF_ERR_INVALID_ARGUMENT);
    pk.offs.push_back(static_cast<int64_t>(pk.tok.size()));
    pk.adv.push_back(0.0);
    const float* tab = upload_table(c.table, policy, c.s);
    rf_batch b{};
    fill_batch(b, c, pk, tab, V, false);
    const double* d_lp = token_logp(c, c.lp, b);
    std::vector<double> lp(pk.tok.size());
    cuda_ok(cudaMemcpyAsync(lp.data(), d_lp, lp.size() * 8, cudaMemcpyDeviceToHost, c.s));
    cuda_ok(cudaStreamSynchronize(c.s));
    TrajectoryRatio out;
    double log_sum = 0.0;
    for (size_t t = 0; t < lp.size(); ++t) {
        const double lr = lp[t] - traj.behavior_logp[t];
        if (!std::isfinite(lr)) throw std::invalid_argument("trajectory_ratio: non-finite log ratio");
        out.per_token.push_back(std::exp(lr));
        log_sum += lr;
    }
    out.product = std::exp(log_sum);
    if (!std::isfinite(out.product)) throw std::invalid_argument("trajectory_ratio: non-finite product");  // :77
    return out;
}

LossResult loss_and_grad(const LossConfig& config, const ToyPolicy& policy, const std::vector<Trajectory>& batch,
                         const LossInputs& aux) {
    config.validate();
    if (batch.empty()) raise(RF_ERR_EMPTY_BATCH);  // losses.cpp:140
    const bool needs_prox = config.variant == LossVariant::decoupled_ppo;
    const bool needs_ref = config.variant == LossVariant::grpo && config.kl_weight > 0.0;
    if (needs_prox && aux.prox == nullptr) raise(RF_ERR_MISSING_PROX);  // :142-144
    if (needs_ref && aux.ref == nullptr) raise(RF_ERR_MISSING_REF);     // :145-148
    if (aux.sg_anchor != nullptr && aux.sg_anchor != &policy)
        throw std::invalid_argument("loss_and_grad: sg_anchor other than the policy is not supported on the GPU path");
    const int C = policy.contexts(), V = policy.vocab();
    const bool cap = config.engine_mismatch_cap > 0.0;
    Packed pk;
    std::vector<std::vector<int32_t>> by_ctx(static_cast<size_t>(C));
    for (size_t i = 0; i < batch.size(); ++i) {
        const Trajectory& t = batch[i];
        if (t.tokens.empty()) raise(RF_ERR_EMPTY_TRAJECTORY);                                       // :157
        if (cap && t.engine_logp.size() != t.tokens.size()) raise(RF_ERR_MISSING_ENGINE_LOGP);    // :173-174
        if (t.context < 0 || t.context >= C) raise(RF_ERR_INVALID_ARGUMENT);
        for (size_t k = 0; k < t.tokens.size(); ++k) {
            if (t.tokens[k] < 0 || t.tokens[k] >= V) raise(RF_ERR_TOKEN_OUT_OF_RANGE);
            by_ctx[static_cast<size_t>(t.context)].push_back(static_cast<int32_t>(pk.tok.size()));
            pk.tok.push_back(t.tokens[k]);
            pk.rows.push_back(t.context);
            pk.sot.push_back(static_cast<int32_t>(i));
            pk.beh.push_back(t.behavior_logp.at(k));
            if (cap) pk.eng.push_back(t.engine_logp[k]);
        }
        pk.offs.push_back(static_cast<int64_t>(pk.tok.size()));
        pk.adv.push_back(t.advantage);
    }
    const size_t T = pk.tok.size();
    Ctx& c = ctx();
    rf_batch b{};
    fill_batch(b, c, pk, upload_table(c.table, policy, c.s), V, cap);
    if (needs_prox) {
        rf_batch q = b;
        q.logits = upload_table(c.prox, *aux.prox, c.s);
        b.prox_logp = token_logp(c, c.lq, q);  // stays on the device
    }
    if (needs_ref) {
        b.ref_logits = upload_table(c.ref, *aux.ref, c.s);
        b.ref_row_stride = V;
    }
    const rf_loss_config cfg = to_c(config);
    rf_outputs o{};
    o.dlogits = c.dl.get<float>(T * static_cast<size_t>(V));
    o.dlogits_dtype = RF_DTYPE_F32;
    o.dlogits_row_stride = V;
    attach_common(o, c, cfg, b);
    rf_status s = rf_loss_and_grad(&cfg, &b, &o, c.s);
    if (s != RF_OK) raise(s);
    // LossResult.grad: per-context fp64 sums of the per-token dlogits rows, in token order
    std::vector<int64_t> segoffs{0};
    std::vector<int32_t> segrows;
    for (const auto& v : by_ctx) {
        segrows.insert(segrows.end(), v.begin(), v.end());
        segoffs.push_back(static_cast<int64_t>(segrows.size()));
    }
    double* d_grad = c.grad.get<double>(static_cast<size_t>(C) * V);
    s = rf_rows_segment_sum(o.dlogits, RF_DTYPE_F32, V, c.segoffs.put(segoffs.data(), segoffs.size(), c.s),
                            c.segrows.put(segrows.data(), segrows.size(), c.s), C, V, d_grad, V, c.s);
    if (s != RF_OK) raise(s);
    LossResult res;
    res.grad.resize(static_cast<size_t>(C) * V);
    double scal[RF_NUM_SCALARS];
    int32_t st = 0;
    cuda_ok(cudaMemcpyAsync(res.grad.data(), d_grad, res.grad.size() * 8, cudaMemcpyDeviceToHost, c.s));
    cuda_ok(cudaMemcpyAsync(scal, o.scalars, sizeof(scal), cudaMemcpyDeviceToHost, c.s));
    cuda_ok(cudaMemcpyAsync(&st, o.device_status, 4, cudaMemcpyDeviceToHost, c.s));
    cuda_ok(cudaStreamSynchronize(c.s));  // also keeps the host vectors alive for the uploads
    if (st & RF_DEVSTAT_NONFINITE_RATIO) raise(RF_ERR_NONFINITE_RATIO);  // losses.cpp:205,267
    if (st & RF_DEVSTAT_TOKEN_OUT_OF_RANGE) raise(RF_ERR_TOKEN_OUT_OF_RANGE);
    if (st & RF_DEVSTAT_EMPTY_TRAJECTORY) raise(RF_ERR_EMPTY_TRAJECTORY);
    res.value = scal[RF_SCALAR_LOSS];
    return res;
}

}  // namespace rlsim
