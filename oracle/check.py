"""Sampled-row parity of a benchmark step against the C oracle (TEST INFRASTRUCTURE ONLY).

bench.py's ``--check K`` leg runs this AFTER its timed region: K token rows of
the last timed step (their logits rows, tokens, advantages and log-prob inputs
exactly as the device saw them) go through ``rf_oracle.c`` and the device's
per-token outputs and dlogits rows are held to the north-star tolerances
(BASELINE.md §5):

* lp, ratio, coefficient, token loss: 1e-5 relative (lp with a 0.01 floor; a
  sequence_product coefficient adds the sequence's accumulated |Δlp|);
* dlogits: |d − d_ref| ≤ 2e-3·|k_t| + half an ulp of the output dtype;
* flags: bit-exact outside the 1e-6 kink band around the clip boundaries
  (the in-band count is reported).

Semantics checked: /root/reference/proj/src/losses.cpp:137-331 via rf_oracle.c.
"""
from __future__ import annotations

import math

import numpy as np

from .pyoracle import oracle_loss_and_grad

REL = 1e-5
DL_ABS = 2e-3
KINK = 1e-6


def kink_band(cfg, lp, b, q, e, seq_offsets) -> np.ndarray:
    """Tokens whose (sequence) log-ratio lies within KINK of a clip boundary."""
    lr = lp - b
    lrq = None if q is None else lp - q
    if int(cfg.aggregation) == 1:
        seq = np.repeat(np.arange(len(seq_offsets) - 1), np.diff(seq_offsets))
        LR = np.bincount(seq, lr, minlength=len(seq_offsets) - 1)
        lr = LR[seq]
        if lrq is not None:
            lrq = np.bincount(seq, lrq, minlength=len(seq_offsets) - 1)[seq]
    v = int(cfg.variant)
    bounds = []
    if v in (0, 5):
        bounds = [(lr, 1 - cfg.clip_eps), (lr, 1 + cfg.clip_eps)]
    elif v == 1 and lrq is not None:
        bounds = [(lrq, 1 - cfg.clip_eps), (lrq, 1 + cfg.clip_eps)]
    elif v in (2, 4):
        bounds = [(lr, cfg.trunc_cap)]
    elif v == 3:
        bounds = [(lr, 1 - cfg.eps_low), (lr, 1 + cfg.eps_high)]
    band = np.zeros(len(lp), dtype=bool)
    for x, bnd in bounds:
        if bnd > 0:
            band |= np.abs(x - math.log(bnd)) < KINK
    if cfg.engine_mismatch_cap > 0 and e is not None:
        band |= np.abs((b - e) - math.log(cfg.engine_mismatch_cap)) < KINK
    return band


def check_sample(cfg, *, logits, token_ids, seq_offsets, advantages, behavior_logp, prox_logp, engine_logp,
                 ref_logits, normalization, global_num_seqs, global_num_tokens, gpu, dl_rows, out_bf16=True,
                 grad_sign=1.0) -> dict:
    """logits [n, V] fp64 (one row per sampled token); gpu = dict of the device's per-token
    outputs for the same tokens (lp, ratio, coef, loss, flags); dl_rows = {i: dlogits row}
    for the sampled tokens whose dlogits row is still on the device.  Returns stats with
    ``ok`` True when every tolerance holds."""
    ref = oracle_loss_and_grad(cfg, logits, token_ids, seq_offsets, advantages, behavior_logp, prox_logp=prox_logp,
                               engine_logp=engine_logp, ref_logits=ref_logits, normalization=normalization,
                               global_num_seqs=global_num_seqs, global_num_tokens=global_num_tokens,
                               grad_sign=grad_sign, want_dlogits=bool(dl_rows))
    band = kink_band(cfg, ref["token_logp"], behavior_logp, prox_logp, engine_logp, seq_offsets)
    ok = ~band
    n = len(token_ids)
    st = {"tokens": int(n), "dlogit_rows": len(dl_rows), "kink_band_tokens": int(band.sum()),
          "oracle_status": int(ref["status"])}

    def rel(a, b, mask, floor):
        if not mask.any():
            return 0.0
        return float((np.abs(a[mask] - b[mask]) / np.maximum(np.abs(b[mask]), floor)).max())

    st["lp_rel"] = rel(gpu["lp"], ref["token_logp"], ok, 1e-2)
    st["ratio_rel"] = rel(gpu["ratio"], ref["token_ratio"], ok, 1e-12)
    tol = np.full(n, REL)
    if int(cfg.aggregation) == 1:
        seq = np.repeat(np.arange(len(seq_offsets) - 1), np.diff(seq_offsets))
        E = np.bincount(seq, np.where(ok, np.abs(gpu["lp"] - ref["token_logp"]), 0.0),
                        minlength=len(seq_offsets) - 1)
        tol = REL + 2.0 * E[seq]
    cm = ok & (ref["token_coef"] != 0)
    cerr = np.abs(gpu["coef"] - ref["token_coef"]) / np.maximum(np.abs(ref["token_coef"]), 1e-300)
    st["coef_rel"] = float(cerr[cm].max()) if cm.any() else 0.0
    coef_ok = bool((cerr[cm] <= tol[cm]).all()) and np.array_equal(gpu["coef"][ok] == 0, ref["token_coef"][ok] == 0)
    scale_l = max(float(np.abs(ref["token_loss"]).max()), 1e-300)
    lerr = np.abs(gpu["loss"] - ref["token_loss"])
    st["token_loss_err"] = float(lerr[ok].max() / scale_l) if ok.any() else 0.0
    loss_ok = bool((lerr[ok] <= REL * scale_l + (tol - REL)[ok] * np.abs(ref["token_loss"][ok])).all())
    flags_ok = np.array_equal(gpu["flags"][ok], ref["token_flags"][ok])
    st["flag_mismatch"] = int((gpu["flags"][ok] != ref["token_flags"][ok]).sum())
    st["flag_mismatch_in_band"] = int((gpu["flags"][band] != ref["token_flags"][band]).sum())
    dl_ok = True
    unit = 0.0
    for i, d in dl_rows.items():
        if band[i]:
            continue
        R = ref["dlogits"][i]
        k = abs(ref["token_coef"][i])
        if int(cfg.variant) == 5 and cfg.kl_weight > 0:
            k = max(k, float(np.abs(R).max()))
        half_ulp = (2.0 ** -8) * np.abs(R) if out_bf16 else 1e-7 * np.abs(R)
        err = np.abs(np.asarray(d, np.float64) - R)
        if (err > DL_ABS * k + half_ulp + 1e-30).any():
            dl_ok = False
        unit = max(unit, float((np.maximum(err - half_ulp, 0) / max(k, 1e-300)).max()))
    st["dlogit_unit_err"] = unit
    st["ok"] = bool(st["lp_rel"] <= REL and st["ratio_rel"] <= REL and coef_ok and loss_ok and flags_ok and dl_ok
                    and ref["status"] == 0)
    return st
