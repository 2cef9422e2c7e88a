// rf_api.cpp — C ABI of include/rf_offpolicy.h: host-side validation mirroring the
// reference's throw sites (losses.cpp:32-39,140-174), kernel selection, cluster
// geometry, and the host-buffer streaming entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "rf_kernels.h"
#include "rf_offpolicy.h"

using rf::KParams;

namespace {

thread_local int32_t g_last_launches = 0;

bool is_aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

struct RingGeometry {
    bool ok = false;
    int kind = 2;  // 2 lag (K2), 3 lag + exact-KL reference row (K2kl)
    int cs = 1, ncw = 0, nvt = 0;
    int row_vecs = 0, slice_vecs = 0, nchunks = 0, nslots = 0;
    size_t smem = 0;
};

int max_optin_smem() {
    static int v = -1;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (v < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 0;
    }
    return v;
}

size_t dtype_size(int32_t d) { return d == RF_DTYPE_BF16 ? 2 : (d == RF_DTYPE_F32 ? 4 : 8); }

// The lag kernel (K2) needs every logits row (and dlogits row) to start on a
// 16-byte boundary with its 16-byte-padded length inside the row stride.  The row
// slice of each CTA lives in registers: pick the smallest cluster whose slice fits
// 12 consumer warps x NVT vectors, then the smallest NVT instance.
RingGeometry ring_geometry(const rf_batch* b, const rf_outputs* o) {
    RingGeometry g;
    const size_t es = dtype_size(b->logits_dtype), os = dtype_size(o->dlogits_dtype);
    const int epv = static_cast<int>(16 / es);
    g.row_vecs = (b->vocab + epv - 1) / epv;
    if (!is_aligned(b->logits, 16) || (b->logits_row_stride * static_cast<int64_t>(es)) % 16 != 0) return g;
    if (b->logits_row_stride < static_cast<int64_t>(g.row_vecs) * epv) return g;
    if (o->dlogits == nullptr || !is_aligned(o->dlogits, 16)) return g;
    if ((o->dlogits_row_stride * static_cast<int64_t>(os)) % 16 != 0) return g;
    if (o->dlogits_row_stride < static_cast<int64_t>(g.row_vecs) * epv) return g;
    g.kind = 2;
    const int ncw = rf::kRingWarpsLag, nct = ncw * 32;
    const size_t tail = rf::kRingLagTailBytes + rf::kRingLagBarrierBytes;
    for (int cs = 1; cs <= 8; cs *= 2) {
        const int slice = (g.row_vecs + cs - 1) / cs;
        if (cs > 1 && slice * (cs - 1) >= g.row_vecs) break;  // every rank must own >= 1 vector
        int nvt = 0;
        for (int q : rf::kRingNvtLag)
            if (static_cast<int64_t>(q) * nct >= slice) {
                nvt = q;
                break;
            }
        if (!nvt) continue;
        const size_t cb = static_cast<size_t>(nct) * rf::lag_vpc(nvt) * 16;
        g.cs = cs;
        g.ncw = ncw;
        g.nvt = nvt;
        g.slice_vecs = slice;
        g.nchunks = static_cast<int>((slice + cb / 16 - 1) / (cb / 16));
        // [nslots x (chunk + full/empty barriers)] + row barriers + tail words
        g.nslots = static_cast<int>((static_cast<size_t>(max_optin_smem()) - tail) / (cb + 16));
        g.smem = static_cast<size_t>(g.nslots) * (cb + 16) + tail;
        g.ok = g.nslots >= 2;
        return g;
    }
    return g;
}

// Exact-KL lag kernel: bf16 policy and reference rows (both 16-byte aligned rows),
// the smallest cluster whose slice fits 12 warps x NVT vectors of each row; every
// ring slot holds a chunk of both rows.
RingGeometry ring_geometry_kl(const rf_batch* b, const rf_outputs* o) {
    RingGeometry g;
    g.kind = 3;
    if (b->logits_dtype != RF_DTYPE_BF16 || !b->ref_logits) return g;
    g.row_vecs = (b->vocab + 7) / 8;
    if (!is_aligned(b->logits, 16) || (b->logits_row_stride * 2) % 16 != 0) return g;
    if (!is_aligned(b->ref_logits, 16) || (b->ref_row_stride * 2) % 16 != 0) return g;
    if (b->logits_row_stride < static_cast<int64_t>(g.row_vecs) * 8) return g;
    if (b->ref_row_stride < static_cast<int64_t>(g.row_vecs) * 8) return g;
    const size_t os = dtype_size(o->dlogits_dtype);
    if (o->dlogits == nullptr || !is_aligned(o->dlogits, 16)) return g;
    if ((o->dlogits_row_stride * static_cast<int64_t>(os)) % 16 != 0) return g;
    if (o->dlogits_row_stride < static_cast<int64_t>(g.row_vecs) * 8) return g;
    const int ncw = rf::kRingWarpsLag, nct = ncw * 32;
    const size_t tail = rf::kRingKLTailBytes + rf::kRingLagBarrierBytes;
    for (int cs = 1; cs <= 8; ++cs) {  // any cluster size: the slice must fit the registers
        const int slice = (g.row_vecs + cs - 1) / cs;
        if (cs > 1 && slice * (cs - 1) >= g.row_vecs) break;
        int nvt = 0;
        for (int q : rf::kRingNvtKL)
            if (static_cast<int64_t>(q) * nct >= slice) {
                nvt = q;
                break;
            }
        if (!nvt) continue;
        const size_t cb = static_cast<size_t>(nct) * rf::lag_vpc(nvt) * 16;
        g.cs = cs;
        g.ncw = ncw;
        g.nvt = nvt;
        g.slice_vecs = slice;
        g.nchunks = static_cast<int>((slice + cb / 16 - 1) / (cb / 16));
        g.nslots = static_cast<int>((static_cast<size_t>(max_optin_smem()) - tail) / (2 * cb + 16));
        g.smem = static_cast<size_t>(g.nslots) * (2 * cb + 16) + tail;
        g.ok = g.nslots >= 2;
        return g;
    }
    return g;
}

int ring_clusters(bool ib, bool ob, int kind, int ncw, int nvt, int cs, size_t smem) {
    struct Key {
        bool ib, ob;
        int kind, ncw, nvt, cs;
        size_t smem;
        int val;
    };
    static std::vector<Key> cache;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    for (const Key& k : cache)
        if (k.ib == ib && k.ob == ob && k.kind == kind && k.ncw == ncw && k.nvt == nvt && k.cs == cs &&
            k.smem == smem)
            return k.val;
    int n = 0;
    const cudaError_t e = kind == 3 ? rf::ring_kl_max_clusters(ob, nvt, cs, smem, &n)
                                    : rf::ring_lag_max_clusters(ib, ob, ncw, nvt, cs, smem, &n);
    if (e != cudaSuccess || n <= 0) {
        cudaGetLastError();
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        n = sms / cs;
    }
    cache.push_back({ib, ob, kind, ncw, nvt, cs, smem, n});
    return n;
}

// exact KL: CTA groups exchanging through L2 (rf_ring_kl.cu GX) fill all 148 SMs
// where 4-CTA hardware clusters place on 132; RF_KL_GX=0 selects the clusters (A/B).
constexpr int kKlMaxGroups = 256;
constexpr size_t kKlSlotBytes = rf::kKlGroupXchBytes;  // per group (rf_kernels.h)
bool kl_groups_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RF_KL_GX");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

int generic_grid(int64_t T) { return static_cast<int>(std::min<int64_t>(T, rf::kGenericMaxGrid)); }

// partial rows: one per token for the lag kernels (per CTA / per sequence elsewhere),
// plus the finalize's scratch rows
int64_t partial_rows(const rf_batch* b) {
    return std::max<int64_t>(std::max<int64_t>(rf::kGenericMaxGrid, b->num_seqs), b->num_tokens) +
           rf::kFinalizeBlocks;
}

// Lag and stream kernels: dynamic row claims (default) or the static walk (RF_ROW_SCHED=static, A/B).
bool dynamic_rows_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RF_ROW_SCHED");
        return !(e && std::string(e) == "static");
    }();
    return on;
}

struct WsLayout {
    double* partials = nullptr;
    double *lse = nullptr, *lp = nullptr, *coef = nullptr, *klx = nullptr, *lseq = nullptr;
    void* xch = nullptr;  // exact-KL CTA-group exchange slots
    unsigned int* row_ctr = nullptr;  // dynamic row counters (lag kernel, or stats + write streams)
    size_t bytes = 0;
};

WsLayout ws_layout(const rf_loss_config* c, const rf_batch* b, void* base) {
    WsLayout w;
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t off = 0;
    auto take = [&](size_t n) {
        void* r = p ? p + off : nullptr;
        off += (n + 255) & ~size_t(255);
        return static_cast<double*>(r);
    };
    w.partials = take(static_cast<size_t>(partial_rows(b)) * RF_NUM_SCALARS * sizeof(double));
    if (c->variant == RF_GRPO && c->kl_weight > 0.0) w.xch = take(kKlMaxGroups * kKlSlotBytes);
    w.row_ctr = reinterpret_cast<unsigned int*>(take(256));
    if (c->aggregation == RF_SEQUENCE_PRODUCT) {
        const size_t T = static_cast<size_t>(b->num_tokens);
        w.lse = take(T * 8);
        w.lp = take(T * 8);
        w.coef = take(T * 8);
        w.klx = take(T * 8);
        w.lseq = take(T * 8);
    }
    w.bytes = off;
    return w;
}

rf_status check_cuda(cudaError_t e) { return e == cudaSuccess ? RF_OK : RF_ERR_CUDA; }

// Per-phase cycle counters of the lag kernel (profiling aid): enabled by the
// environment variable RF_DEBUG_COUNTERS=1, read with rf_debug_counters().
unsigned long long* debug_counters() {
    static unsigned long long* buf = nullptr;
    static int enabled = -1;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (enabled < 0) {
        const char* e = std::getenv("RF_DEBUG_COUNTERS");
        enabled = (e && e[0] == '1') ? 1 : 0;
        if (enabled && cudaMalloc(&buf, rf::kDbgWords * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(buf, 0, rf::kDbgWords * sizeof(unsigned long long));
        else
            buf = nullptr;
    }
    return buf;
}

}  // namespace

extern "C" {

void rf_loss_config_default(rf_loss_config* c) {
    c->variant = RF_PPO;
    c->aggregation = RF_TOKEN_MEAN;
    c->clip_eps = 0.2;
    c->eps_low = 0.2;
    c->eps_high = 0.2;
    c->trunc_cap = 5.0;
    c->kl_weight = 0.0;
    c->w_plus = 1.0;
    c->w_minus = 1.0;
    c->engine_mismatch_cap = 0.0;
}

rf_status rf_loss_config_validate(const rf_loss_config* c) {
    if (!c) return RF_ERR_INVALID_ARGUMENT;
    if (!(c->clip_eps > 0.0 && c->clip_eps < 1.0)) return RF_ERR_CLIP_EPS;
    if (c->eps_low < 0.0 || c->eps_high < 0.0) return RF_ERR_EPS_LOW_HIGH;
    if (c->trunc_cap <= 0.0) return RF_ERR_TRUNC_CAP;
    if (c->kl_weight < 0.0) return RF_ERR_KL_WEIGHT;
    if (c->w_plus < 0.0 || c->w_minus < 0.0) return RF_ERR_TOPR_WEIGHTS;
    if (c->engine_mismatch_cap < 0.0) return RF_ERR_MISMATCH_CAP;
    if (c->variant < RF_PPO || c->variant > RF_NAIVE_IS) return RF_ERR_UNKNOWN_VARIANT;
    if (c->aggregation != RF_TOKEN_MEAN && c->aggregation != RF_SEQUENCE_PRODUCT) return RF_ERR_INVALID_ARGUMENT;
    return RF_OK;
}

const char* rf_loss_variant_name(int32_t v) {
    switch (v) {
        case RF_PPO: return "ppo";
        case RF_DECOUPLED_PPO: return "decoupled_ppo";
        case RF_TIS: return "tis";
        case RF_CISPO: return "cispo";
        case RF_TOPR: return "topr";
        case RF_GRPO: return "grpo";
        case RF_NAIVE_IS: return "naive_is";
    }
    return "unknown";
}

rf_status rf_loss_variant_from_name(const char* name, int32_t* out) {
    if (!name || !out) return RF_ERR_INVALID_ARGUMENT;
    for (int32_t v = RF_PPO; v <= RF_NAIVE_IS; ++v) {
        if (std::strcmp(name, rf_loss_variant_name(v)) == 0) {
            *out = v;
            return RF_OK;
        }
    }
    return RF_ERR_UNKNOWN_VARIANT;
}

const char* rf_status_string(rf_status s) {
    switch (s) {
        case RF_OK: return "ok";
        case RF_ERR_CLIP_EPS: return "LossConfig: clip_eps must be in (0,1)";
        case RF_ERR_EPS_LOW_HIGH: return "LossConfig: eps_low/eps_high must be >= 0";
        case RF_ERR_TRUNC_CAP: return "LossConfig: trunc_cap must be > 0";
        case RF_ERR_KL_WEIGHT: return "LossConfig: kl_weight must be >= 0";
        case RF_ERR_TOPR_WEIGHTS: return "LossConfig: TOPR weights must be >= 0";
        case RF_ERR_MISMATCH_CAP: return "LossConfig: engine_mismatch_cap must be >= 0";
        case RF_ERR_EMPTY_BATCH: return "loss_and_grad: empty batch";
        case RF_ERR_MISSING_PROX: return "loss_and_grad: decoupled_ppo requires a proximal policy";
        case RF_ERR_MISSING_REF: return "loss_and_grad: grpo with kl_weight > 0 requires a reference policy";
        case RF_ERR_EMPTY_TRAJECTORY: return "loss_and_grad: empty trajectory";
        case RF_ERR_MISSING_ENGINE_LOGP: return "loss_and_grad: engine log-probs missing for mismatch correction";
        case RF_ERR_NONFINITE_RATIO: return "loss_and_grad: non-finite ratio";
        case RF_ERR_GROUP_TOO_SMALL: return "grpo_advantages: group size must be >= 2";
        case RF_ERR_UNKNOWN_VARIANT: return "unknown loss variant";
        case RF_ERR_INVALID_ARGUMENT: return "invalid argument";
        case RF_ERR_UNSUPPORTED_LAYOUT: return "unsupported layout";
        case RF_ERR_TOKEN_OUT_OF_RANGE: return "token id out of range";
        case RF_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
        case RF_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

size_t rf_workspace_bytes(const rf_loss_config* c, const rf_batch* b) {
    if (!c || !b) return 0;
    return ws_layout(c, b, nullptr).bytes;
}

int32_t rf_last_launch_count(void) { return g_last_launches; }

int32_t rf_debug_counters(uint64_t* out, int32_t n, int32_t reset) {
    unsigned long long* buf = debug_counters();
    if (!buf || !out || n <= 0) return 0;
    n = n > rf::kDbgWords ? rf::kDbgWords : n;
    cudaDeviceSynchronize();
    cudaMemcpy(out, buf, static_cast<size_t>(n) * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    if (reset) cudaMemset(buf, 0, rf::kDbgWords * sizeof(unsigned long long));
    return n;
}

rf_status rf_zero_scalars(rf_outputs* o, void* stream) {
    if (!o || !o->scalars || !o->device_status) return RF_ERR_INVALID_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(o->scalars, 0, RF_NUM_SCALARS * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(o->device_status, 0, sizeof(int32_t), st);
    return check_cuda(e);
}

rf_status rf_grpo_advantages(const rf_batch* b, rf_outputs* o, void* stream) {
    if (!b || !o) return RF_ERR_INVALID_ARGUMENT;
    if (b->num_groups <= 0) return RF_ERR_EMPTY_BATCH;
    if (!b->rewards || !b->group_offsets || !o->advantages_out || !o->group_degenerate || !o->device_status)
        return RF_ERR_INVALID_ARGUMENT;
    g_last_launches = 1;
    return check_cuda(rf::launch_grpo(b->rewards, b->group_offsets, b->num_groups, o->advantages_out,
                                      o->group_degenerate, o->device_status, static_cast<cudaStream_t>(stream)));
}

rf_status rf_loss_and_grad_ex(const rf_loss_config* c, const rf_batch* b, rf_outputs* o, void* stream,
                              int32_t kernel) {
    g_last_launches = 0;
    if (!c || !b || !o) return RF_ERR_INVALID_ARGUMENT;
    rf_status st = rf_loss_config_validate(c);
    if (st != RF_OK) return st;
    if (b->num_tokens <= 0 || b->num_seqs <= 0) return RF_ERR_EMPTY_BATCH;            // losses.cpp:140
    const bool needs_prox = c->variant == RF_DECOUPLED_PPO;
    const bool needs_ref = c->variant == RF_GRPO && c->kl_weight > 0.0;
    if (needs_prox && !b->prox_logp) return RF_ERR_MISSING_PROX;                       // losses.cpp:142-144
    if (needs_ref && !b->ref_logits) return RF_ERR_MISSING_REF;                        // losses.cpp:145-148
    if (c->engine_mismatch_cap > 0.0 && !b->engine_logp) return RF_ERR_MISSING_ENGINE_LOGP;  // losses.cpp:173
    if (!b->logits || !b->token_ids || !b->seq_of_token || !b->seq_offsets || !b->advantages || !b->behavior_logp)
        return RF_ERR_INVALID_ARGUMENT;
    if (!o->scalars || !o->device_status) return RF_ERR_INVALID_ARGUMENT;
    if (b->vocab < 2) return RF_ERR_INVALID_ARGUMENT;
    if (b->logits_dtype != RF_DTYPE_BF16 && b->logits_dtype != RF_DTYPE_F32) return RF_ERR_INVALID_ARGUMENT;
    if (o->dlogits && o->dlogits_dtype != RF_DTYPE_BF16 && o->dlogits_dtype != RF_DTYPE_F32)
        return RF_ERR_INVALID_ARGUMENT;
    if (b->logp_dtype != RF_DTYPE_F32 && b->logp_dtype != RF_DTYPE_F64) return RF_ERR_INVALID_ARGUMENT;
    if (b->normalization == RF_NORM_SEQ_THEN_BATCH && b->global_num_seqs <= 0) return RF_ERR_INVALID_ARGUMENT;
    if (b->normalization == RF_NORM_GLOBAL_TOKEN && b->global_num_tokens <= 0) return RF_ERR_INVALID_ARGUMENT;
    if (b->normalization != RF_NORM_SEQ_THEN_BATCH && b->normalization != RF_NORM_GLOBAL_TOKEN)
        return RF_ERR_INVALID_ARGUMENT;
    if (b->logits_row_stride < b->vocab) return RF_ERR_INVALID_ARGUMENT;
    if (needs_ref && b->ref_row_stride < b->vocab) return RF_ERR_INVALID_ARGUMENT;
    if (o->dlogits && o->dlogits_row_stride < b->vocab) return RF_ERR_INVALID_ARGUMENT;

    const WsLayout ws = ws_layout(c, b, o->workspace);
    if (!o->workspace || o->workspace_bytes < ws.bytes) return RF_ERR_WORKSPACE_TOO_SMALL;

    KParams p{};
    p.variant = c->variant;
    p.aggregation = c->aggregation;
    p.clip_eps = c->clip_eps;
    p.eps_low = c->eps_low;
    p.eps_high = c->eps_high;
    p.trunc_cap = c->trunc_cap;
    p.kl_weight = c->kl_weight;
    p.w_plus = c->w_plus;
    p.w_minus = c->w_minus;
    p.mismatch_cap = c->engine_mismatch_cap;
    p.T = b->num_tokens;
    p.V = b->vocab;
    p.logp_f64 = b->logp_dtype == RF_DTYPE_F64 ? 1 : 0;
    p.logits = b->logits;
    p.row_stride = b->logits_row_stride;
    p.ref_logits = needs_ref ? b->ref_logits : nullptr;
    p.ref_row_stride = b->ref_row_stride;
    p.row_of_token = b->row_of_token;
    p.token_ids = b->token_ids;
    p.seq_of_token = b->seq_of_token;
    p.seq_offsets = b->seq_offsets;
    p.advantages = b->advantages;
    p.behavior_logp = b->behavior_logp;
    p.prox_logp = b->prox_logp;
    p.engine_logp = b->engine_logp;
    p.normalization = b->normalization;
    p.inv_n = b->global_num_seqs > 0 ? 1.0 / static_cast<double>(b->global_num_seqs) : 0.0;
    p.inv_t = b->global_num_tokens > 0 ? 1.0 / static_cast<double>(b->global_num_tokens) : 0.0;
    p.grad_sign = b->grad_sign;
    p.dlogits = o->dlogits;
    p.dl_stride = o->dlogits_row_stride;
    p.token_logp = o->token_logp;
    p.token_ratio = o->token_ratio;
    p.token_coef = o->token_coef;
    p.token_loss = o->token_loss;
    p.token_flags = o->token_flags;
    p.status = o->device_status;
    p.partials = ws.partials;
    p.mode = 0;
    p.dbg = debug_counters();

    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool ib = b->logits_dtype == RF_DTYPE_BF16;
    const bool ob = o->dlogits_dtype == RF_DTYPE_BF16;
    int64_t nparts = 0;

    if (c->aggregation == RF_SEQUENCE_PRODUCT) {
        // Two passes over the logits (losses.cpp:180-259): the sequence weights
        // need every token's log-prob first.
        p.tok_lse = ws.lse;
        p.tok_klx = ws.klx;
        p.tok_lseq = ws.lseq;
        p.token_logp = o->token_logp ? o->token_logp : ws.lp;
        const int grid = generic_grid(b->num_tokens);
        p.mode = 1;
        // Fast path (ring-compatible layout): K2st, the read-only online-softmax stats
        // stream (lse per token, one read of the logits), the sequence scalars, then the
        // K2w dlogits stream — 6·V bytes per token.  Exact KL and unaligned layouts take
        // the generic kernel.
        RingGeometry g;
        if (kernel != RF_KERNEL_GENERIC && !needs_ref) g = ring_geometry(b, o);
        if (kernel == RF_KERNEL_RING && !g.ok) return RF_ERR_UNSUPPORTED_LAYOUT;
        if (g.ok) {
            p.row_vecs = g.row_vecs;
            // dynamic row claims (stats stream: counter 0, write stream: counter 1)
            if (dynamic_rows_enabled()) {
                p.row_ctr = ws.row_ctr;
                if (cudaMemsetAsync(ws.row_ctr, 0, 2 * sizeof(unsigned int), s) != cudaSuccess) return RF_ERR_CUDA;
            }
            if (rf::launch_stream_stats(p, ib, s) != cudaSuccess) return RF_ERR_CUDA;
        } else {
            if (rf::launch_generic(p, ib, ob, grid, s) != cudaSuccess) return RF_ERR_CUDA;
        }
        if (rf::launch_seq(p, 0, b->num_seqs, ws.coef, s) != cudaSuccess) return RF_ERR_CUDA;
        if (o->token_coef)
            if (cudaMemcpyAsync(o->token_coef, ws.coef, static_cast<size_t>(b->num_tokens) * 8,
                                cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                return RF_ERR_CUDA;
        nparts = b->num_seqs;
        g_last_launches = 2;
        if (o->dlogits) {
            KParams q = p;
            q.mode = 2;
            q.token_coef = ws.coef;
            if (q.row_ctr) q.row_ctr += 1;
            const cudaError_t e = g.ok ? rf::launch_stream_write(q, ib, ob, s) : rf::launch_generic(q, ib, ob, grid, s);
            if (e != cudaSuccess) return RF_ERR_CUDA;
            g_last_launches += 1;
        }
    } else {
        RingGeometry g;
        if (kernel != RF_KERNEL_GENERIC) g = needs_ref ? ring_geometry_kl(b, o) : ring_geometry(b, o);
        if (kernel == RF_KERNEL_RING && !g.ok) return RF_ERR_UNSUPPORTED_LAYOUT;
        if (g.ok) {
            p.slice_vecs = g.slice_vecs;
            p.row_vecs = g.row_vecs;
            p.nchunks = g.nchunks;
            p.nslots = g.nslots;
            int maxc = ring_clusters(ib, ob, g.kind, g.ncw, g.nvt, g.cs, g.smem);
            if (g.kind == 3 && g.cs > 1 && kl_groups_enabled()) {
                int dev = 0, sms = 148;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                maxc = std::min(kKlMaxGroups, sms / g.cs);
                p.vcs = g.cs;
                p.xch = ws.xch;
                // The groups' L2 exchange slots carry sequence words row + 1: zero them in
                // stream order before every launch, so no slot of an earlier launch (or an
                // earlier replay of a captured CUDA graph) can match.
                if (cudaMemsetAsync(ws.xch, 0, static_cast<size_t>(kKlMaxGroups) * kKlSlotBytes, s) != cudaSuccess)
                    return RF_ERR_CUDA;
            }
            // the lag kernels write one partial row per token: scalars independent of which
            // cluster took which row (bit-identical with static and dynamic row claims)
            p.row_ctr = nullptr;
            if (dynamic_rows_enabled()) {
                p.row_ctr = ws.row_ctr;
                if (cudaMemsetAsync(ws.row_ctr, 0, sizeof(unsigned int), s) != cudaSuccess) return RF_ERR_CUDA;
            }
            int ncl = static_cast<int>(std::min<int64_t>(b->num_tokens, maxc));
            cudaError_t e = g.kind == 3 ? rf::launch_ring_kl(p, ob, g.nvt, g.cs, ncl, g.smem, s)
                                        : rf::launch_ring_lag(p, ib, ob, g.ncw, g.nvt, g.cs, ncl, g.smem, s);
            if (e == cudaErrorCooperativeLaunchTooLarge && p.vcs > 0) {
                // the CTA groups need every CTA co-resident (e.g. SMs held by an MPS
                // partition): the hardware-cluster version instead
                cudaGetLastError();
                p.vcs = 0;
                ncl = static_cast<int>(
                    std::min<int64_t>(b->num_tokens, ring_clusters(ib, ob, g.kind, g.ncw, g.nvt, g.cs, g.smem)));
                e = rf::launch_ring_kl(p, ob, g.nvt, g.cs, ncl, g.smem, s);
            }
            if (e != cudaSuccess) return RF_ERR_CUDA;
            nparts = b->num_tokens;  // lag kernels: one partial row per token
        } else {
            const int grid = generic_grid(b->num_tokens);
            if (rf::launch_generic(p, ib, ob, grid, s) != cudaSuccess) return RF_ERR_CUDA;
            nparts = grid;
        }
        g_last_launches = 1;
    }
    if (rf::launch_finalize(ws.partials, nparts, o->scalars, b->seq_of_token, b->seq_offsets, b->num_tokens,
                            b->num_seqs, o->device_status, s) != cudaSuccess)
        return RF_ERR_CUDA;
    g_last_launches += rf::finalize_launches(nparts);
    return RF_OK;
}

rf_status rf_lmhead_lse(const void* hidden, const void* w_vocab, const int32_t* token_ids, int64_t num_tokens,
                        int32_t vocab, int32_t hidden_dim, double* lse, float* x_tok, void* stream) {
    if (!hidden || !w_vocab || !token_ids || !lse || !x_tok) return RF_ERR_INVALID_ARGUMENT;
    if (num_tokens <= 0) return RF_ERR_EMPTY_BATCH;
    if (vocab < 2 || hidden_dim <= 0 || hidden_dim % 64 != 0) return RF_ERR_INVALID_ARGUMENT;
    if (!is_aligned(hidden, 16) || !is_aligned(w_vocab, 16)) return RF_ERR_UNSUPPORTED_LAYOUT;
    const cudaError_t e = rf::launch_lmhead_lse(hidden, w_vocab, token_ids, num_tokens, vocab, hidden_dim, lse, x_tok,
                                                static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return RF_ERR_CUDA;
    g_last_launches = 1;
    return RF_OK;
}

rf_status rf_lmhead_dlogits(const void* hidden, const void* w_vocab, const int32_t* token_ids, int64_t num_tokens,
                            int32_t vocab, int32_t hidden_dim, const double* lse, const double* coef, void* dlogits,
                            int64_t dlogits_row_stride, void* stream) {
    if (!hidden || !w_vocab || !token_ids || !lse || !coef || !dlogits) return RF_ERR_INVALID_ARGUMENT;
    if (num_tokens <= 0) return RF_ERR_EMPTY_BATCH;
    if (vocab < 2 || hidden_dim <= 0 || hidden_dim % 64 != 0 || dlogits_row_stride < vocab)
        return RF_ERR_INVALID_ARGUMENT;
    if (!is_aligned(hidden, 16) || !is_aligned(w_vocab, 16) || !is_aligned(dlogits, 16) ||
        (dlogits_row_stride * 2) % 16 != 0)
        return RF_ERR_UNSUPPORTED_LAYOUT;
    const cudaError_t e = rf::launch_lmhead_dlogits(hidden, w_vocab, token_ids, num_tokens, vocab, hidden_dim, lse, coef,
                                                    dlogits, dlogits_row_stride, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return RF_ERR_CUDA;
    g_last_launches = 1;
    return RF_OK;
}

rf_status rf_token_loss_from_stats(const rf_loss_config* c, const rf_batch* b, const double* lse, const float* x_tok,
                                   rf_outputs* o, void* stream) {
    g_last_launches = 0;
    if (!c || !b || !o || !lse || !x_tok) return RF_ERR_INVALID_ARGUMENT;
    rf_status st = rf_loss_config_validate(c);
    if (st != RF_OK) return st;
    if (b->num_tokens <= 0 || b->num_seqs <= 0) return RF_ERR_EMPTY_BATCH;
    if (c->aggregation != RF_TOKEN_MEAN || (c->variant == RF_GRPO && c->kl_weight > 0.0))
        return RF_ERR_INVALID_ARGUMENT;  // token_mean without exact KL (a per-token row sum is not available here)
    if (c->variant == RF_DECOUPLED_PPO && !b->prox_logp) return RF_ERR_MISSING_PROX;
    if (c->engine_mismatch_cap > 0.0 && !b->engine_logp) return RF_ERR_MISSING_ENGINE_LOGP;
    if (!b->token_ids || !b->seq_of_token || !b->seq_offsets || !b->advantages || !b->behavior_logp)
        return RF_ERR_INVALID_ARGUMENT;
    if (!o->scalars || !o->device_status) return RF_ERR_INVALID_ARGUMENT;
    if (b->logp_dtype != RF_DTYPE_F32 && b->logp_dtype != RF_DTYPE_F64) return RF_ERR_INVALID_ARGUMENT;
    if (b->normalization == RF_NORM_SEQ_THEN_BATCH && b->global_num_seqs <= 0) return RF_ERR_INVALID_ARGUMENT;
    if (b->normalization == RF_NORM_GLOBAL_TOKEN && b->global_num_tokens <= 0) return RF_ERR_INVALID_ARGUMENT;
    const WsLayout ws = ws_layout(c, b, o->workspace);
    if (!o->workspace || o->workspace_bytes < ws.bytes) return RF_ERR_WORKSPACE_TOO_SMALL;
    KParams p{};
    p.variant = c->variant;
    p.aggregation = c->aggregation;
    p.clip_eps = c->clip_eps;
    p.eps_low = c->eps_low;
    p.eps_high = c->eps_high;
    p.trunc_cap = c->trunc_cap;
    p.kl_weight = c->kl_weight;
    p.w_plus = c->w_plus;
    p.w_minus = c->w_minus;
    p.mismatch_cap = c->engine_mismatch_cap;
    p.T = b->num_tokens;
    p.V = b->vocab;
    p.logp_f64 = b->logp_dtype == RF_DTYPE_F64 ? 1 : 0;
    p.token_ids = b->token_ids;
    p.seq_of_token = b->seq_of_token;
    p.seq_offsets = b->seq_offsets;
    p.advantages = b->advantages;
    p.behavior_logp = b->behavior_logp;
    p.prox_logp = b->prox_logp;
    p.engine_logp = b->engine_logp;
    p.normalization = b->normalization;
    p.inv_n = b->global_num_seqs > 0 ? 1.0 / static_cast<double>(b->global_num_seqs) : 0.0;
    p.inv_t = b->global_num_tokens > 0 ? 1.0 / static_cast<double>(b->global_num_tokens) : 0.0;
    p.grad_sign = b->grad_sign;
    p.token_logp = o->token_logp;
    p.token_ratio = o->token_ratio;
    p.token_coef = o->token_coef;
    p.token_loss = o->token_loss;
    p.token_flags = o->token_flags;
    p.status = o->device_status;
    p.partials = ws.partials;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (rf::launch_token_loss(p, lse, x_tok, s) != cudaSuccess) return RF_ERR_CUDA;
    if (rf::launch_finalize(ws.partials, (b->num_tokens + 255) / 256, o->scalars, b->seq_of_token, b->seq_offsets,
                            b->num_tokens, b->num_seqs, o->device_status, s) != cudaSuccess)
        return RF_ERR_CUDA;
    g_last_launches = 1 + rf::finalize_launches((b->num_tokens + 255) / 256);
    return RF_OK;
}

rf_status rf_rows_segment_sum(const void* rows, int32_t rows_dtype, int64_t row_stride, const int64_t* seg_offsets,
                              const int32_t* seg_rows, int64_t num_segments, int32_t width, double* out,
                              int64_t out_stride, void* stream) {
    if (!rows || !seg_offsets || !seg_rows || !out) return RF_ERR_INVALID_ARGUMENT;
    if (rows_dtype != RF_DTYPE_BF16 && rows_dtype != RF_DTYPE_F32) return RF_ERR_INVALID_ARGUMENT;
    if (num_segments <= 0 || width <= 0 || row_stride < width || out_stride < width) return RF_ERR_INVALID_ARGUMENT;
    if (num_segments > 65535) return RF_ERR_UNSUPPORTED_LAYOUT;
    g_last_launches = 1;
    return check_cuda(rf::launch_rows_segment_sum(rows, rows_dtype == RF_DTYPE_BF16, row_stride, seg_offsets, seg_rows,
                                                  num_segments, width, out, out_stride,
                                                  static_cast<cudaStream_t>(stream)));
}

rf_status rf_loss_and_grad(const rf_loss_config* c, const rf_batch* b, rf_outputs* o, void* stream) {
    return rf_loss_and_grad_ex(c, b, o, stream, RF_KERNEL_AUTO);
}

}  // extern "C"
