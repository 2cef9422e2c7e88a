"""GPU parity in the regime the benchmark runs: many rows per CTA / cluster.

The persistent kernels walk many rows per CTA (or cluster) — claimed from a per-launch
counter, or c, c + ncl, c + 2·ncl, … with RF_ROW_SCHED=static — so everything that only
exists from the second row on — the lag kernel's
row-to-row TMEM parking, the even/odd scalar warps, the bar_red/bar_bc phase
alternation, the xslot[row & 3] exchange slots, ring-slot phase flips, the
stream kernels' double-buffered per-row slots, the exact-KL CTA groups' L2
sequence words, the host API's double-buffered chunks — is exercised only when
T ≫ the number of CTAs.  Every case here has ≥ 16 rows per CTA / cluster
(T ≥ 2,368 at V = 32,000 over 148 CTAs; T ≥ 1,184 at V = 151,936 over 74
2-CTA clusters), rows drawn through a wrapping ``row_of_token`` pool as in
bench.py's DeviceWorkload, and compares EVERY token's lp / ratio / coefficient /
loss / flags with the fp64 oracle (semantics: reference losses.cpp:137-331) plus
the dlogits of ~64 sampled rows including the first and last row of several
clusters.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from tests.cases import VARIANTS, config, make_pool_case
from tests.parity import DL_ABS, compare, run_oracle, to_device_batch

pytestmark = pytest.mark.gpu

import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import _abi  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402

SMS = 148


def _cfg(v, **kw):
    return config(v, engine_mismatch_cap=kw.pop("cap", 2.0), **kw)


def sampled_rows(T, ncl, n_random=48, seed=0):
    """First and last row of clusters 0, 1, ncl/2, ncl-1, plus random rows."""
    sel = set()
    for c in {0, 1, ncl // 2, ncl - 1}:
        if c < T:
            sel.add(c)
            sel.add(c + ((T - 1 - c) // ncl) * ncl)
    rng = np.random.default_rng(seed)
    sel.update(rng.choice(T, size=min(n_random, T), replace=False).tolist())
    return np.array(sorted(sel))


def check_dlogit_rows(case, cfg, gpu, ref, rows, out_dtype=torch.bfloat16):
    """dlogits of the sampled rows against k_t·(onehot − p) from the oracle's coefficient
    and its fp64 log-softmax of the row (LogProbGrad add/flush, losses.cpp:87-115)."""
    D = gpu.dlogits[torch.from_numpy(rows).to(gpu.dlogits.device)].double().cpu().numpy()
    worst = 0.0
    for i, t in enumerate(rows):
        r = int(case.row_of_token[t]) if case.row_of_token is not None else int(t)
        p = np.exp(O.oracle_log_softmax(case.logits[r]))
        k = float(ref["token_coef"][t])
        R = -(k * p)
        tok = int(case.token_ids[t])
        R[tok] = k - k * p[tok]
        if k == 0.0:
            R[:] = 0.0
        half = (2.0 ** -8) * np.abs(R) if out_dtype == torch.bfloat16 else 1e-7 * np.abs(R)
        err = np.abs(D[i] - R)
        assert (err <= DL_ABS * abs(k) + half + 1e-30).all(), (t, float((err - half).max() / max(abs(k), 1e-300)))
        worst = max(worst, float((np.maximum(err - half, 0) / max(abs(k), 1e-300)).max()))
    return worst


def check_kl_dlogit_rows(case, cfg, gpu, rows, T_global):
    """Exact-KL rows: the oracle on the sampled tokens alone (mapping A, 1/T_global per
    token, so each token's coefficient and KL term are the full batch's)."""
    r = case.row_of_token[rows]
    sub = O.oracle_loss_and_grad(cfg, case.logits[r], case.token_ids[rows], np.arange(len(rows) + 1),
                                 case.advantages[np.searchsorted(case.seq_offsets, rows, side="right") - 1],
                                 case.behavior_logp[rows], prox_logp=case.prox_logp[rows],
                                 engine_logp=case.engine_logp[rows], ref_logits=case.ref_logits[r], normalization=1,
                                 global_num_tokens=T_global)
    D = gpu.dlogits[torch.from_numpy(rows).to(gpu.dlogits.device)].double().cpu().numpy()
    R = sub["dlogits"]
    k = np.maximum(np.abs(sub["token_coef"])[:, None], np.abs(R).max(axis=1, keepdims=True))
    half = (2.0 ** -8) * np.abs(R)
    err = np.abs(D - R)
    assert (err <= DL_ABS * k + half + 1e-30).all(), float(((err - half) / k).max())


# ---------------------------------------------------------------------------
# K2 ring_lag_kernel: Qwen3 vocab, 74 two-CTA clusters, ~28 rows per cluster
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def qwen3_pool():
    return make_pool_case(101, V=151936, R=192, T_min=16 * (SMS // 2) + 900, G=8, max_len=96, stale=0.25,
                          alpha=2)


@pytest.mark.parametrize("variant", VARIANTS)
def test_ring_lag_many_rows_per_cluster_qwen3(qwen3_pool, variant):
    case = qwen3_pool
    assert case.T >= 16 * (SMS // 2)
    cfg = _cfg(variant)
    norm = L.Normalization.global_token
    pb = to_device_batch(case, normalization=norm)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=int(norm), want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, SMS // 2, seed=VARIANTS.index(variant)))


# ---------------------------------------------------------------------------
# V = 32,000: one CTA per row, 148 CTAs, ~28 rows per CTA
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def v32k_pool():
    return make_pool_case(102, V=32000, R=384, T_min=16 * SMS + 1800, G=8, max_len=128, stale=0.25, alpha=8)


@pytest.mark.parametrize("variant", VARIANTS)
def test_ring_lag_many_rows_per_cta_v32k(v32k_pool, variant):
    case = v32k_pool
    assert case.T >= 16 * SMS
    cfg = _cfg(variant)
    norm = L.Normalization.global_token
    pb = to_device_batch(case, normalization=norm)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=int(norm), want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, SMS, seed=7 + VARIANTS.index(variant)))


@pytest.mark.parametrize("variant", ["ppo", "tis"])
def test_generic_kernel_many_rows(v32k_pool, variant):
    """The generic kernel's persistent grid (≤ 1,184 CTAs) also walks several rows each."""
    case = v32k_pool
    cfg = _cfg(variant)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel="generic")
    ref = run_oracle(case, cfg, normalization=1, want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, 8 * SMS, n_random=16))


@pytest.mark.parametrize("variant", ["ppo", "decoupled_ppo", "tis"])
def test_ring_lag_mapping_b_many_rows(variant):
    """Rows shared per sequence (the reference layout, 1/(N·L_i)) at many rows per CTA."""
    case = make_pool_case(103, V=32000, R=97, T_min=16 * SMS + 500, G=4, max_len=64, stale=0.25, mapping="B")
    cfg = _cfg(variant)
    pb = to_device_batch(case)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=0, want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, SMS, n_random=32))


@pytest.mark.parametrize("variant", ["tis", "decoupled_ppo"])
def test_ring_lag_f32_logits_cluster4_many_rows(variant):
    """f32 rows of 151,936 span 4-CTA clusters (37 of them): ~28 rows per cluster."""
    case = make_pool_case(104, V=151936, R=64, T_min=16 * (SMS // 4) + 450, G=4, max_len=48, stale=0.2,
                          round_bf16=False)
    case.logits = case.logits.astype(np.float32).astype(np.float64)
    cfg = _cfg(variant)
    pb = to_device_batch(case, dtype=torch.float32, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, dlogits_dtype=torch.float32, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1, want_dlogits=False)
    compare(case, cfg, gpu, ref, out_dtype=torch.float32, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, SMS // 4, n_random=24), out_dtype=torch.float32)


# ---------------------------------------------------------------------------
# sequence_product: K2st / K2s / K2w stream kernels, T > 3 x their grid
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("variant", ["ppo", "decoupled_ppo", "tis", "cispo", "topr", "naive_is"])
def test_stream_kernels_many_rows_v32k(v32k_pool, variant):
    case = v32k_pool
    assert case.T > 3 * 8 * SMS
    cfg = _cfg(variant, aggregation="sequence_product")
    pb = to_device_batch(case, normalization=L.Normalization.seq_then_batch)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=0, want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, 8 * SMS, n_random=48))


@pytest.mark.parametrize("variant", ["tis", "decoupled_ppo"])
def test_stream_kernels_many_rows_qwen3(variant):
    case = make_pool_case(105, V=151936, R=128, T_min=3 * 8 * SMS + 600, G=8, max_len=64, stale=0.05)
    cfg = _cfg(variant, aggregation="sequence_product")
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1, want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gpu, ref, sampled_rows(case.T, 8 * SMS, n_random=40))


# ---------------------------------------------------------------------------
# exact KL: 37 CTA groups of 4 over L2, ~28 rows per group
# ---------------------------------------------------------------------------
def test_grpo_kl_many_rows_per_group():
    case = make_pool_case(106, V=151936, R=96, T_min=16 * (SMS // 4) + 450, G=4, max_len=48, stale=0.2, kl=True)
    cfg = _cfg("grpo", kl_weight=0.1)
    pb = to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1, want_dlogits=False)
    compare(case, cfg, gpu, ref, check_dlogits=False)
    check_kl_dlogit_rows(case, cfg, gpu, sampled_rows(case.T, SMS // 4, n_random=24), case.T)
    again = rf.loss_and_grad(cfg, pb, kernel="ring")
    assert torch.equal(gpu.dlogits, again.dlogits)


# ---------------------------------------------------------------------------
# rf_loss_and_grad_host: >= 8 double-buffered chunks, bit-equal to the device API
# ---------------------------------------------------------------------------
def _host_call(case, cfg, chunk, norm):
    """rf_loss_and_grad_host on pinned host buffers with one logits row per token."""
    V = case.V
    rows = case.row_of_token
    pool = torch.from_numpy(case.logits).to(torch.bfloat16)
    h_logits = torch.empty(case.T, V, dtype=torch.bfloat16).pin_memory()
    h_logits.copy_(pool[torch.from_numpy(rows).long()])
    h_dl = torch.zeros(case.T, V, dtype=torch.bfloat16).pin_memory()
    pin = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dt).pin_memory()
    h_tok = pin(case.token_ids, torch.int32)
    h_offs = pin(case.seq_offsets, torch.int64)
    h_seq = pin(np.repeat(np.arange(case.N), np.diff(case.seq_offsets)), torch.int32)
    h_adv = pin(case.advantages, torch.float64)
    h_b, h_q, h_e = (pin(a, torch.float64) for a in (case.behavior_logp, case.prox_logp, case.engine_logp))
    outs = {k: torch.zeros(case.T, dtype=torch.float64).pin_memory() for k in ["lp", "ratio", "coef", "loss"]}
    h_flags = torch.zeros(case.T, dtype=torch.uint8).pin_memory()
    h_scal = torch.zeros(_abi.RF_NUM_SCALARS, dtype=torch.float64).pin_memory()
    h_status = torch.zeros(1, dtype=torch.int32).pin_memory()
    b = _abi.rf_batch()
    b.num_tokens, b.num_seqs, b.vocab = case.T, case.N, V
    b.logits_dtype, b.logits, b.logits_row_stride = _abi.RF_DTYPE_BF16, h_logits.data_ptr(), V
    b.token_ids, b.seq_of_token, b.seq_offsets = h_tok.data_ptr(), h_seq.data_ptr(), h_offs.data_ptr()
    b.advantages = h_adv.data_ptr()
    b.logp_dtype, b.normalization = _abi.RF_DTYPE_F64, int(norm)
    b.behavior_logp, b.prox_logp, b.engine_logp = h_b.data_ptr(), h_q.data_ptr(), h_e.data_ptr()
    b.global_num_seqs, b.global_num_tokens, b.grad_sign = case.N, case.T, 1.0
    o = _abi.rf_outputs()
    o.dlogits, o.dlogits_dtype, o.dlogits_row_stride = h_dl.data_ptr(), _abi.RF_DTYPE_BF16, V
    o.token_logp, o.token_ratio = outs["lp"].data_ptr(), outs["ratio"].data_ptr()
    o.token_coef, o.token_loss, o.token_flags = outs["coef"].data_ptr(), outs["loss"].data_ptr(), h_flags.data_ptr()
    o.scalars, o.device_status = h_scal.data_ptr(), h_status.data_ptr()
    c = cfg.to_c()
    st = _abi.load_library().rf_loss_and_grad_host(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), 0, chunk)
    assert st == 0, L.status_string(st)
    return outs, h_flags, h_dl, h_scal


@pytest.mark.parametrize("variant,agg", [("decoupled_ppo", "token_mean"), ("cispo", "token_mean"),
                                         ("tis", "sequence_product")])
def test_host_api_many_chunks_bit_equal_device(variant, agg):
    chunk = 512
    case = make_pool_case(107, V=151936, R=160, T_min=9 * chunk + 100, G=4, max_len=160, stale=0.1)
    cfg = _cfg(variant, aggregation=agg)
    norm = L.Normalization.global_token if agg == "token_mean" else L.Normalization.seq_then_batch
    outs, flags, h_dl, scal = _host_call(case, cfg, chunk, norm)
    assert case.T >= 8 * chunk
    pb = to_device_batch(case, normalization=norm)
    dev = rf.loss_and_grad(cfg, pb, kernel="auto")
    # per-token outputs and dlogits bit-equal to one device call over the pooled rows
    assert np.array_equal(outs["lp"].numpy(), dev.token_logp.cpu().numpy())
    assert np.array_equal(outs["ratio"].numpy(), dev.token_ratio.cpu().numpy())
    assert np.array_equal(outs["coef"].numpy(), dev.token_coef.cpu().numpy())
    assert np.array_equal(outs["loss"].numpy(), dev.token_loss.cpu().numpy())
    assert np.array_equal(flags.numpy(), dev.token_flags.cpu().numpy())
    assert torch.equal(h_dl, dev.dlogits.cpu())
    sc, sd = scal.numpy(), dev.scalars.cpu().numpy()
    assert abs(sc[0] - sd[0]) <= 1e-12 * max(1.0, abs(sd[0]))
    assert np.array_equal(sc[1:6], sd[1:6])
    # and the host call against the oracle
    ref = run_oracle(case, cfg, normalization=int(norm), want_dlogits=False)

    class R:
        pass

    gr = R()
    gr.token_logp, gr.token_ratio, gr.token_coef = (torch.from_numpy(outs[k].numpy()) for k in ("lp", "ratio", "coef"))
    gr.token_loss, gr.token_flags, gr.scalars, gr.dlogits = (torch.from_numpy(outs["loss"].numpy()), flags,
                                                             scal, h_dl)
    compare(case, cfg, gr, ref, check_dlogits=False)
    check_dlogit_rows(case, cfg, gr, ref, sampled_rows(case.T, chunk, n_random=32))


# ---------------------------------------------------------------------------
# Row schedule: dynamic row claims (default) vs the static walk c, c + ncl, ...
# (RF_ROW_SCHED=static, read once per process: a subprocess).  The per-row math and the
# per-token partial rows do not depend on which cluster took a row, so the two are
# bit-identical — scalars, token outputs and dlogits.
# ---------------------------------------------------------------------------
_SCHED_ARM = """
import sys
sys.path.insert(0, {root!r})
import torch
import paper_2510_11345_b200 as rf
from tests.test_gpu_bench_regime import _sched_case
cfg, pb = _sched_case({kl!r})
r = rf.loss_and_grad(cfg, pb, kernel="ring")
torch.save({{k: getattr(r, k).cpu() for k in _FIELDS}}, {out!r})
print("arm ok")
""".replace("_FIELDS", repr(["scalars", "dlogits", "token_logp", "token_ratio", "token_coef", "token_loss",
                             "token_flags"]))


def _sched_case(kl):
    if kl == "seqprod":  # the sequence_product stats / write streams (up to 1,184 CTAs, ~4 rows each)
        case = make_pool_case(109, V=32000, R=256, T_min=4 * 8 * SMS + 300, G=8, max_len=160, stale=0.25, alpha=4)
        cfg = _cfg("tis", aggregation="sequence_product")
        return cfg, to_device_batch(case, normalization=L.Normalization.seq_then_batch)
    if kl:
        case = make_pool_case(107, V=151936, R=96, T_min=16 * (SMS // 4) + 300, G=4, max_len=48, stale=0.2, kl=True)
        cfg = _cfg("grpo", kl_weight=0.1)
        return cfg, to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    case = make_pool_case(108, V=151936, R=128, T_min=16 * (SMS // 2) + 500, G=8, max_len=96, stale=0.25, alpha=2)
    cfg = _cfg("decoupled_ppo")
    return cfg, to_device_batch(case, normalization=L.Normalization.global_token)


@pytest.mark.parametrize("kl", [False, True, "seqprod"])
def test_row_schedule_static_bit_equal_dynamic(kl, tmp_path):
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "static.pt")
    r = subprocess.run([sys.executable, "-c", _SCHED_ARM.format(root=root, kl=kl, out=out)],
                       env={**os.environ, "RF_ROW_SCHED": "static"}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "arm ok" in r.stdout, r.stdout + r.stderr
    static = torch.load(out)
    cfg, pb = _sched_case(kl)
    dyn = rf.loss_and_grad(cfg, pb, kernel="ring")
    for k, v in static.items():
        assert torch.equal(getattr(dyn, k).cpu(), v), k
