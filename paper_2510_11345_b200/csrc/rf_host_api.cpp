// rf_host_api.cpp — rf_loss_and_grad_host: the reference-facing call with HOST
// buffers (the shape of rlsim::loss_and_grad, losses.cpp:137: host logits in,
// host gradient + value out).  Validates like the reference (every throw site of
// losses.cpp:32-39,140-174, empty trajectories, token ids), then streams the batch
// through the GPU in token chunks with three streams:
//   h2d:     logits chunk i+1 (pinned host -> device ring buffer)
//   compute: rf_loss_and_grad on chunk i
//   d2h:     dlogits chunk i-1 (device -> host)
// so PCIe traffic in both directions overlaps the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "rf_offpolicy.h"

namespace {

size_t dsz(int32_t d) { return d == RF_DTYPE_BF16 ? 2 : (d == RF_DTYPE_F32 ? 4 : 8); }

struct Chunk {
    int64_t t0, t1;  // token range
    int64_t s0, s1;  // sequence range (sequence_product: the call's sub-view)
};

// The host API's own stream-ordered memory pool per device, with its memory kept
// mapped between calls (a release threshold of 0 would return it to the OS at every
// synchronisation).  Private, so the process's default pool (e.g. PyTorch's
// cudaMallocAsync backend) keeps its own trimming behaviour.
cudaMemPool_t host_api_pool(int device) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(device);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[device] = pool;
    return pool;
}

struct DevBuf {
    void* p = nullptr;
    cudaMemPool_t pool = nullptr;
    cudaError_t alloc(size_t n, cudaStream_t s) { return n ? cudaMallocFromPoolAsync(&p, n, pool, s) : cudaSuccess; }
    void release(cudaStream_t s) {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
    }
};

}  // namespace

extern "C" rf_status rf_loss_and_grad_host(const rf_loss_config* c, const rf_batch* hb, rf_outputs* ho,
                                           int32_t device, int64_t chunk_tokens) {
    if (!c || !hb || !ho) return RF_ERR_INVALID_ARGUMENT;
    rf_status st = rf_loss_config_validate(c);
    if (st != RF_OK) return st;
    const int64_t T = hb->num_tokens, N = hb->num_seqs;
    if (T <= 0 || N <= 0) return RF_ERR_EMPTY_BATCH;
    if (c->variant == RF_DECOUPLED_PPO && !hb->prox_logp) return RF_ERR_MISSING_PROX;
    if (c->variant == RF_GRPO && c->kl_weight > 0.0 && !hb->ref_logits) return RF_ERR_MISSING_REF;
    if (c->engine_mismatch_cap > 0.0 && !hb->engine_logp) return RF_ERR_MISSING_ENGINE_LOGP;
    if (!hb->logits || !hb->token_ids || !hb->seq_of_token || !hb->seq_offsets || !hb->advantages ||
        !hb->behavior_logp || !ho->scalars)
        return RF_ERR_INVALID_ARGUMENT;
    // Host-side validation the device path cannot afford.
    if (hb->seq_offsets[N] - hb->seq_offsets[0] != T) return RF_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < N; ++i)
        if (hb->seq_offsets[i + 1] <= hb->seq_offsets[i]) return RF_ERR_EMPTY_TRAJECTORY;  // losses.cpp:157
    for (int64_t t = 0; t < T; ++t)
        if (hb->token_ids[t] < 0 || hb->token_ids[t] >= hb->vocab) return RF_ERR_TOKEN_OUT_OF_RANGE;
    int64_t table_rows = 0;
    if (hb->row_of_token) {
        for (int64_t t = 0; t < T; ++t) {
            if (hb->row_of_token[t] < 0) return RF_ERR_INVALID_ARGUMENT;
            table_rows = std::max<int64_t>(table_rows, hb->row_of_token[t] + 1);
        }
    }
    if (cudaSetDevice(device) != cudaSuccess) return RF_ERR_CUDA;

    const bool seqprod = c->aggregation == RF_SEQUENCE_PRODUCT;
    const bool kl = c->variant == RF_GRPO && c->kl_weight > 0.0;
    if (chunk_tokens <= 0) chunk_tokens = 16384;
    // Chunks: token ranges for token_mean; whole-sequence ranges for sequence_product.
    std::vector<Chunk> chunks;
    if (!seqprod) {
        for (int64_t t = 0; t < T; t += chunk_tokens) chunks.push_back({t, std::min(T, t + chunk_tokens), 0, N});
    } else {
        int64_t s = 0;
        while (s < N) {
            int64_t e = s + 1;
            while (e < N && hb->seq_offsets[e + 1] - hb->seq_offsets[s] <= chunk_tokens) ++e;
            chunks.push_back({hb->seq_offsets[s] - hb->seq_offsets[0], hb->seq_offsets[e] - hb->seq_offsets[0], s, e});
            s = e;
        }
    }
    int64_t max_chunk = 0;
    for (const Chunk& ch : chunks) max_chunk = std::max(max_chunk, ch.t1 - ch.t0);

    const size_t les = dsz(hb->logits_dtype), des = dsz(ho->dlogits_dtype), lps = dsz(hb->logp_dtype);
    const bool per_token_rows = hb->row_of_token == nullptr;
    const size_t row_bytes = static_cast<size_t>(hb->logits_row_stride) * les;
    const size_t drow_bytes = static_cast<size_t>(ho->dlogits_row_stride) * des;

    cudaMemPool_t pool = host_api_pool(device);
    if (!pool) return RF_ERR_CUDA;
    cudaStream_t s_h2d, s_cmp, s_d2h;
    cudaStreamCreateWithFlags(&s_h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s_cmp, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s_d2h, cudaStreamNonBlocking);
    cudaEvent_t ev_in[2], ev_cmp[2], ev_out[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_cmp[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming);
    }

    // Metadata + per-token outputs (whole batch), logits/dlogits chunk double buffers.
    DevBuf d_tok, d_seqof, d_offs, d_adv, d_b, d_q, d_e, d_rows, d_table, d_ref, d_lin[2], d_dout[2], d_lp, d_ratio,
        d_coef, d_loss, d_flags, d_scal, d_status, d_ws;
    rf_status rc = RF_OK;
    auto A = [&](DevBuf& b, size_t n) {
        b.pool = pool;
        if (rc == RF_OK && b.alloc(n, s_cmp) != cudaSuccess) rc = RF_ERR_CUDA;
    };
    A(d_tok, T * 4);
    A(d_seqof, T * 4);
    A(d_offs, (N + 1) * 8);
    A(d_adv, N * 8);
    A(d_b, T * lps);
    if (hb->prox_logp) A(d_q, T * lps);
    if (hb->engine_logp) A(d_e, T * lps);
    if (!per_token_rows) {
        A(d_rows, T * 4);
        A(d_table, static_cast<size_t>(table_rows) * row_bytes);
        if (kl) A(d_ref, static_cast<size_t>(table_rows) * hb->ref_row_stride * les);
    } else {
        for (int i = 0; i < 2; ++i) A(d_lin[i], static_cast<size_t>(max_chunk) * row_bytes);
        if (kl) A(d_ref, static_cast<size_t>(T) * hb->ref_row_stride * les);
    }
    if (ho->dlogits)
        for (int i = 0; i < 2; ++i) A(d_dout[i], static_cast<size_t>(max_chunk) * drow_bytes);
    if (ho->token_logp) A(d_lp, T * 8);
    if (ho->token_ratio) A(d_ratio, T * 8);
    if (ho->token_coef) A(d_coef, T * 8);
    if (ho->token_loss) A(d_loss, T * 8);
    if (ho->token_flags) A(d_flags, T);
    A(d_scal, RF_NUM_SCALARS * 8);
    A(d_status, 4);
    rf_batch probe = *hb;
    probe.num_tokens = max_chunk;
    probe.num_seqs = N;
    const size_t wsb = rf_workspace_bytes(c, &probe);
    A(d_ws, wsb);

    auto H2D = [&](void* dst, const void* src, size_t n, cudaStream_t s) {
        if (rc == RF_OK && n && cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s) != cudaSuccess)
            rc = RF_ERR_CUDA;
    };
    H2D(d_tok.p, hb->token_ids, T * 4, s_cmp);
    // sequence_product calls see a sub-view of the sequence arrays, so each chunk's
    // seq_of_token is rebased to its first sequence (host copy, uploaded once)
    std::vector<int32_t> rebased;
    if (seqprod) {
        rebased.resize(static_cast<size_t>(T));
        for (const Chunk& ch : chunks)
            for (int64_t t = ch.t0; t < ch.t1; ++t)
                rebased[static_cast<size_t>(t)] = hb->seq_of_token[t] - static_cast<int32_t>(ch.s0);
    }
    H2D(d_seqof.p, seqprod ? rebased.data() : static_cast<const void*>(hb->seq_of_token), T * 4, s_cmp);
    H2D(d_offs.p, hb->seq_offsets, (N + 1) * 8, s_cmp);
    H2D(d_adv.p, hb->advantages, N * 8, s_cmp);
    H2D(d_b.p, hb->behavior_logp, T * lps, s_cmp);
    if (hb->prox_logp) H2D(d_q.p, hb->prox_logp, T * lps, s_cmp);
    if (hb->engine_logp) H2D(d_e.p, hb->engine_logp, T * lps, s_cmp);
    if (!per_token_rows) {
        H2D(d_rows.p, hb->row_of_token, T * 4, s_cmp);
        H2D(d_table.p, hb->logits, static_cast<size_t>(table_rows) * row_bytes, s_cmp);
        if (kl) H2D(d_ref.p, hb->ref_logits, static_cast<size_t>(table_rows) * hb->ref_row_stride * les, s_cmp);
    } else if (kl) {
        H2D(d_ref.p, hb->ref_logits, static_cast<size_t>(T) * hb->ref_row_stride * les, s_cmp);
    }
    if (rc == RF_OK) {
        cudaMemsetAsync(d_scal.p, 0, RF_NUM_SCALARS * 8, s_cmp);
        cudaMemsetAsync(d_status.p, 0, 4, s_cmp);
    }
    cudaEvent_t ev_meta;
    cudaEventCreateWithFlags(&ev_meta, cudaEventDisableTiming);
    cudaEventRecord(ev_meta, s_cmp);
    cudaStreamWaitEvent(s_h2d, ev_meta, 0);
    cudaStreamWaitEvent(s_d2h, ev_meta, 0);

    for (size_t i = 0; i < chunks.size() && rc == RF_OK; ++i) {
        const Chunk& ch = chunks[i];
        const int bi = static_cast<int>(i & 1);
        const int64_t n = ch.t1 - ch.t0;
        if (per_token_rows) {
            if (i >= 2) cudaStreamWaitEvent(s_h2d, ev_cmp[bi], 0);  // chunk i-2 finished reading d_lin[bi]
            H2D(d_lin[bi].p, static_cast<const uint8_t*>(hb->logits) + static_cast<size_t>(ch.t0) * row_bytes,
                static_cast<size_t>(n) * row_bytes, s_h2d);
            cudaEventRecord(ev_in[bi], s_h2d);
            cudaStreamWaitEvent(s_cmp, ev_in[bi], 0);
        }
        if (ho->dlogits && i >= 2) cudaStreamWaitEvent(s_cmp, ev_out[bi], 0);  // chunk i-2's D2H done

        rf_batch db = *hb;
        db.num_tokens = n;
        db.logits = per_token_rows ? d_lin[bi].p : d_table.p;
        db.row_of_token = per_token_rows ? nullptr : static_cast<const int32_t*>(d_rows.p) + ch.t0;
        db.token_ids = static_cast<const int32_t*>(d_tok.p) + ch.t0;
        db.seq_of_token = static_cast<const int32_t*>(d_seqof.p) + ch.t0;
        db.behavior_logp = static_cast<const uint8_t*>(d_b.p) + ch.t0 * lps;
        db.prox_logp = hb->prox_logp ? static_cast<const uint8_t*>(d_q.p) + ch.t0 * lps : nullptr;
        db.engine_logp = hb->engine_logp ? static_cast<const uint8_t*>(d_e.p) + ch.t0 * lps : nullptr;
        db.ref_logits = kl ? (per_token_rows ? static_cast<const uint8_t*>(d_ref.p) +
                                                   static_cast<size_t>(ch.t0) * hb->ref_row_stride * les
                                             : d_ref.p)
                           : nullptr;
        if (seqprod) {
            // sub-view of the sequence arrays; seq_of_token must index it
            db.num_seqs = ch.s1 - ch.s0;
            db.seq_offsets = static_cast<const int64_t*>(d_offs.p) + ch.s0;
            db.advantages = static_cast<const double*>(d_adv.p) + ch.s0;
        } else {
            db.seq_offsets = static_cast<const int64_t*>(d_offs.p);
            db.advantages = static_cast<const double*>(d_adv.p);
        }
        db.group_offsets = nullptr;
        db.rewards = nullptr;
        rf_outputs dout{};
        dout.dlogits = ho->dlogits ? d_dout[bi].p : nullptr;
        dout.dlogits_dtype = ho->dlogits_dtype;
        dout.dlogits_row_stride = ho->dlogits_row_stride;
        dout.token_logp = ho->token_logp ? static_cast<double*>(d_lp.p) + ch.t0 : nullptr;
        dout.token_ratio = ho->token_ratio ? static_cast<double*>(d_ratio.p) + ch.t0 : nullptr;
        dout.token_coef = ho->token_coef ? static_cast<double*>(d_coef.p) + ch.t0 : nullptr;
        dout.token_loss = ho->token_loss ? static_cast<double*>(d_loss.p) + ch.t0 : nullptr;
        dout.token_flags = ho->token_flags ? static_cast<uint8_t*>(d_flags.p) + ch.t0 : nullptr;
        dout.scalars = static_cast<double*>(d_scal.p);
        dout.device_status = static_cast<int32_t*>(d_status.p);
        dout.workspace = d_ws.p;
        dout.workspace_bytes = wsb;
        const rf_status ks = rf_loss_and_grad(c, &db, &dout, s_cmp);
        if (ks != RF_OK) rc = ks;
        cudaEventRecord(ev_cmp[bi], s_cmp);
        if (ho->dlogits) {
            cudaStreamWaitEvent(s_d2h, ev_cmp[bi], 0);
            if (rc == RF_OK &&
                cudaMemcpyAsync(static_cast<uint8_t*>(ho->dlogits) + static_cast<size_t>(ch.t0) * drow_bytes,
                                d_dout[bi].p, static_cast<size_t>(n) * drow_bytes, cudaMemcpyDeviceToHost,
                                s_d2h) != cudaSuccess)
                rc = RF_ERR_CUDA;
            cudaEventRecord(ev_out[bi], s_d2h);
        }
    }
    cudaStreamSynchronize(s_d2h);
    cudaStreamSynchronize(s_h2d);
    auto D2H = [&](void* dst, const void* src, size_t n) {
        if (rc == RF_OK && dst && n && cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s_cmp) != cudaSuccess)
            rc = RF_ERR_CUDA;
    };
    int32_t dev_status = 0;
    D2H(ho->token_logp, d_lp.p, T * 8);
    D2H(ho->token_ratio, d_ratio.p, T * 8);
    D2H(ho->token_coef, d_coef.p, T * 8);
    D2H(ho->token_loss, d_loss.p, T * 8);
    D2H(ho->token_flags, d_flags.p, T);
    D2H(ho->scalars, d_scal.p, RF_NUM_SCALARS * 8);
    D2H(&dev_status, d_status.p, 4);
    if (cudaStreamSynchronize(s_cmp) != cudaSuccess && rc == RF_OK) rc = RF_ERR_CUDA;
    if (ho->device_status) *ho->device_status = dev_status;

    for (DevBuf* b : {&d_tok, &d_seqof, &d_offs, &d_adv, &d_b, &d_q, &d_e, &d_rows, &d_table, &d_ref, &d_lin[0],
                      &d_lin[1], &d_dout[0], &d_dout[1], &d_lp, &d_ratio, &d_coef, &d_loss, &d_flags, &d_scal,
                      &d_status, &d_ws})
        b->release(s_cmp);
    cudaStreamSynchronize(s_cmp);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(ev_in[i]);
        cudaEventDestroy(ev_cmp[i]);
        cudaEventDestroy(ev_out[i]);
    }
    cudaEventDestroy(ev_meta);
    cudaStreamDestroy(s_h2d);
    cudaStreamDestroy(s_cmp);
    cudaStreamDestroy(s_d2h);
    if (rc == RF_OK && (dev_status & RF_DEVSTAT_NONFINITE_RATIO)) rc = RF_ERR_NONFINITE_RATIO;  // losses.cpp:267
    if (rc == RF_OK && (dev_status & RF_DEVSTAT_TOKEN_OUT_OF_RANGE)) rc = RF_ERR_TOKEN_OUT_OF_RANGE;
    if (rc == RF_OK && (dev_status & RF_DEVSTAT_EMPTY_TRAJECTORY)) rc = RF_ERR_EMPTY_TRAJECTORY;
    return rc;
}
