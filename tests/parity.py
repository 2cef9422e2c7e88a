"""GPU-vs-oracle comparison helpers.

Tolerances (north star, BASELINE.json):
  * per-token log-probs, ratios, coefficients, token losses and the loss value:
    1e-5 relative (fp32 softmax sums, fp64 per-token math);
  * dlogits: 2e-3 absolute on the unit-coefficient dlogit (onehot - p), i.e.
    |d_gpu - d_ref| <= 2e-3 * |k_t|, plus the half-ulp of the output dtype
    (2^-8 relative for bf16) that storing the value in bf16 costs by itself;
  * masks / flags / token counts: bit-exact, except tokens whose log-ratio lies
    within 1e-6 of a clip boundary (the kink band — fp32 vs fp64 softmax can
    legitimately land on either side), which are counted and reported.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np
import torch

import oracle as O
from paper_2510_11345_b200 import losses as L
from paper_2510_11345_b200._abi import RF_FLAG_CLIPPED, RF_FLAG_MISMATCH_CAPPED, RF_FLAG_ZERO_COEF

REL = 1e-5
DL_ABS = 2e-3
KINK = 1e-6


def to_device_batch(case, *, dtype=torch.bfloat16, normalization=L.Normalization.seq_then_batch, pad_to=8,
                    logp_dtype=torch.float64, grad_sign=1.0, global_num_seqs=None, global_num_tokens=None,
                    with_ref=False, device="cuda"):
    V = case.V
    padV = (V + pad_to - 1) // pad_to * pad_to
    lg = torch.zeros(case.logits.shape[0], padV, dtype=dtype, device=device)
    lg[:, :V] = torch.from_numpy(case.logits).to(device=device, dtype=dtype)
    ref = None
    if with_ref and case.ref_logits is not None:
        ref = torch.zeros(case.ref_logits.shape[0], padV, dtype=dtype, device=device)
        ref[:, :V] = torch.from_numpy(case.ref_logits).to(device=device, dtype=dtype)
        ref = ref[:, :V]

    def t(a, dt):
        return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)

    return L.PackedBatch(
        logits=lg[:, :V], token_ids=t(case.token_ids, torch.int32), seq_offsets=t(case.seq_offsets, torch.int64),
        advantages=t(case.advantages, torch.float64), behavior_logp=t(case.behavior_logp, logp_dtype),
        row_of_token=t(case.row_of_token, torch.int32), prox_logp=t(case.prox_logp, logp_dtype),
        engine_logp=t(case.engine_logp, logp_dtype), ref_logits=ref, normalization=normalization,
        global_num_seqs=global_num_seqs, global_num_tokens=global_num_tokens, grad_sign=grad_sign,
        rewards=t(case.rewards, torch.float64), group_offsets=t(case.group_offsets, torch.int64))


def logp_as_seen(case, dt):
    """The per-token log-prob inputs exactly as the device sees them."""
    if dt == torch.float32:
        f = lambda a: None if a is None else np.asarray(a, np.float32).astype(np.float64)
    else:
        f = lambda a: a
    return f(case.behavior_logp), f(case.prox_logp), f(case.engine_logp)


def run_oracle(case, cfg, *, normalization=0, logp_dtype=torch.float64, grad_sign=1.0, want_dlogits=True,
               global_num_seqs=None, global_num_tokens=None, logits=None):
    b, q, e = logp_as_seen(case, logp_dtype)
    return O.oracle_loss_and_grad(
        cfg, case.logits if logits is None else logits, case.token_ids, case.seq_offsets, case.advantages, b,
        prox_logp=q, engine_logp=e, row_of_token=case.row_of_token, ref_logits=case.ref_logits,
        normalization=int(normalization), grad_sign=grad_sign, want_dlogits=want_dlogits,
        global_num_seqs=global_num_seqs, global_num_tokens=global_num_tokens)


def kink_band(case, cfg, ref_out, logp_dtype=torch.float64) -> np.ndarray:
    """Tokens whose (sequence) log-ratio lies within KINK of a clip boundary."""
    b, q, e = logp_as_seen(case, logp_dtype)
    lp = ref_out["token_logp"]
    lr = lp - b
    if int(cfg.aggregation) == 1:
        lens = np.diff(case.seq_offsets)
        seq = np.repeat(np.arange(case.N), lens)
        LR = np.zeros(case.N)
        np.add.at(LR, seq, lr)
        lr = LR[seq]
        if q is not None:
            LPX = np.zeros(case.N)
            np.add.at(LPX, seq, lp - q)
            lrq = LPX[seq]
    else:
        lrq = lp - q if q is not None else None
    bounds = []
    v = int(cfg.variant)
    if v in (0, 5):
        bounds = [(lr, 1 - cfg.clip_eps), (lr, 1 + cfg.clip_eps)]
    elif v == 1:
        bounds = [(lrq, 1 - cfg.clip_eps), (lrq, 1 + cfg.clip_eps), (lr, None)]
    elif v == 2 or v == 4:
        bounds = [(lr, cfg.trunc_cap)]
    elif v == 3:
        bounds = [(lr, 1 - cfg.eps_low), (lr, 1 + cfg.eps_high)]
    band = np.zeros(case.T, dtype=bool)
    for x, bnd in bounds:
        if bnd is None or bnd <= 0:
            continue
        band |= np.abs(x - math.log(bnd)) < KINK
    if v == 1:
        # min-branch tie r*A vs po*c*A
        band |= np.abs(lr - (lrq + 0)) < 0  # no extra tie handling needed beyond the clip edges
    if cfg.engine_mismatch_cap > 0 and e is not None:
        band |= np.abs((b - e) - math.log(cfg.engine_mismatch_cap)) < KINK
    return band


def compare(case, cfg, gpu: L.LossResult, ref: dict, **kw):
    """Assert parity; returns a dict of observed max errors.  With RF_PARITY_LOG=<file>
    the stats of every passing comparison are appended there as JSON lines (precision
    reports across library variants)."""
    stats = _compare(case, cfg, gpu, ref, **kw)
    log = os.environ.get("RF_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], **stats}) + "\n")
    return stats


def _compare(case, cfg, gpu: L.LossResult, ref: dict, *, out_dtype=torch.bfloat16, check_dlogits=True,
             logp_dtype=torch.float64, rows=None):
    band = kink_band(case, cfg, ref, logp_dtype)
    ok = ~band
    stats = {"kink_band_tokens": int(band.sum())}
    g = lambda t: t.detach().double().cpu().numpy()
    lp = g(gpu.token_logp)
    ratio = g(gpu.token_ratio)
    coef = g(gpu.token_coef)
    tloss = g(gpu.token_loss)
    flags = gpu.token_flags.cpu().numpy()

    def rel(a, b, mask, atol=1e-12):
        if not mask.any():
            return 0.0
        d = np.abs(a[mask] - b[mask]) / np.maximum(np.abs(b[mask]), atol)
        return float(d.max())

    stats["lp_rel"] = rel(lp, ref["token_logp"], ok, 1e-2)
    stats["ratio_rel"] = rel(ratio, ref["token_ratio"], ok, 1e-12)
    stats["coef_rel"] = rel(coef, ref["token_coef"], ok & (ref["token_coef"] != 0), 1e-300)
    assert stats["lp_rel"] <= REL, stats
    assert stats["ratio_rel"] <= REL, stats
    # sequence_product: the sequence ratio is exp(Σ_t (lp_t − b_t)) (losses.cpp:187-252), so
    # its relative error is the ABSOLUTE error of the sum — the per-token lp errors (each
    # within REL, checked above) add up along the sequence.  The coefficient and loss
    # tolerance of a token is REL plus twice its sequence's accumulated |Δlp| (LR and LPX
    # both carry it); token_mean keeps the flat REL.
    tol = np.full(case.T, REL)
    if int(cfg.aggregation) == 1:
        lens = np.diff(case.seq_offsets)
        seq = np.repeat(np.arange(case.N), lens)
        E = np.zeros(case.N)
        np.add.at(E, seq, np.where(ok, np.abs(lp - ref["token_logp"]), 0.0))
        tol = REL + 2.0 * E[seq]
        stats["seq_lp_err_max"] = float(E.max())
    cm = ok & (ref["token_coef"] != 0)
    if cm.any():
        d = np.abs(coef[cm] - ref["token_coef"][cm]) / np.abs(ref["token_coef"][cm])
        assert (d <= tol[cm]).all(), stats
    # zero coefficients exactly where the oracle has them (outside the band)
    assert np.array_equal(coef[ok] == 0, ref["token_coef"][ok] == 0), stats
    assert np.array_equal(flags[ok], ref["token_flags"][ok]), (stats, np.nonzero(flags[ok] != ref["token_flags"][ok]))
    stats["flag_mismatch_in_band"] = int((flags[band] != ref["token_flags"][band]).sum())
    # token losses: 1e-5 relative to the largest per-token magnitude (they cancel)
    scale_l = max(np.abs(ref["token_loss"]).max(), 1e-300)
    stats["token_loss_err"] = float(np.abs(tloss[ok] - ref["token_loss"][ok]).max() / scale_l) if ok.any() else 0.0
    if ok.any():
        lb = REL * scale_l + (tol - REL)[ok] * np.abs(ref["token_loss"][ok])
        assert (np.abs(tloss[ok] - ref["token_loss"][ok]) <= lb).all(), stats
    val = float(gpu.scalars[0])
    if not band.any():
        # The value is the sum of the (verified) per-token losses, which cancel — the
        # advantages are zero-mean per group, and the exact-KL penalty offsets the
        # policy term.  Its error is bounded by REL of its own magnitude plus the
        # propagated per-token errors (each within REL, checked above); relative to
        # a floor of 1e-3 of the summed magnitudes that bound is reported as value_rel.
        denom = max(abs(ref["value"]), np.abs(ref["token_loss"]).sum() * 1e-3, 1e-300)
        stats["value_rel"] = abs(val - ref["value"]) / denom
        prop = float(np.abs(tloss - ref["token_loss"]).sum())
        stats["value_err_vs_propagated"] = abs(val - ref["value"]) / max(prop, 1e-300)
        assert abs(val - ref["value"]) <= REL * denom + 2.0 * prop, (stats, val, ref["value"])
    sc = gpu.scalars.cpu().numpy()
    assert int(sc[1]) == case.T
    if not band.any():
        assert int(sc[2]) == int(((ref["token_flags"] & RF_FLAG_CLIPPED) != 0).sum())
        assert int(sc[4]) == int(((ref["token_flags"] & RF_FLAG_ZERO_COEF) != 0).sum())
        assert int(sc[5]) == int(((ref["token_flags"] & RF_FLAG_MISMATCH_CAPPED) != 0).sum())
    if check_dlogits and gpu.dlogits is not None:
        D = g(gpu.dlogits)
        R = ref["dlogits"]
        k = np.abs(ref["token_coef"])[:, None]
        if int(cfg.variant) == 5 and cfg.kl_weight > 0:
            # KL rows carry a second coefficient; scale by the row's magnitude
            k = np.maximum(k, np.abs(R).max(axis=1, keepdims=True))
        half_ulp = (2.0 ** -8) * np.abs(R) if out_dtype == torch.bfloat16 else 1e-7 * np.abs(R)
        err = np.abs(D - R)
        bound = DL_ABS * k + half_ulp + 1e-30
        sel = ok if rows is None else ok & rows
        viol = (err > bound)[sel]
        kk = np.maximum(k, 1e-300)
        stats["dlogit_unit_err"] = float((np.maximum(err - half_ulp, 0) / kk)[sel].max()) if sel.any() else 0.0
        assert not viol.any(), stats
    return stats
