"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref, compiled from
/root/reference by oracle/Makefile).  Run here (needs the reference build):

    python tests/golden/make_golden.py

Writes tests/golden/golden_v1.npz: GRPO groups with the reference's advantages,
loss_and_grad cases (every variant x aggregation x row mapping) with the
reference's value, [C x V] gradient and per-row log-probs, the reference's
RngStream draws, and toy_train_loop learning curves.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from tests.cases import VARIANTS, config, make_case  # noqa: E402


def main():
    O.build()
    assert O.ref_available(), "oracle/_ref not built (needs /root/reference)"
    out = {}
    rng = np.random.default_rng(20251018)
    # --- GRPO groups (losses.cpp:41-60) ---
    sizes = rng.integers(2, 20, 60)
    go = np.zeros(len(sizes) + 1, dtype=np.int64)
    go[1:] = np.cumsum(sizes)
    rewards = rng.uniform(-3, 3, go[-1])
    for g in range(0, len(sizes), 6):
        rewards[go[g]:go[g + 1]] = 0.25  # degenerate groups
    rewards[go[3]:go[4]] = (rng.uniform(0, 1, sizes[3]) < 0.5).astype(float)
    adv = np.zeros_like(rewards)
    deg = np.zeros(len(sizes), dtype=np.uint8)
    for g in range(len(sizes)):
        a, d = O.ref_grpo_advantages(rewards[go[g]:go[g + 1]])
        adv[go[g]:go[g + 1]] = a
        deg[g] = d
    out.update(grpo_rewards=rewards, grpo_offsets=go, grpo_adv=adv, grpo_deg=deg)

    # --- loss_and_grad cases ---
    names = []
    for mapping in ["A", "B"]:
        for agg in ["token_mean", "sequence_product"]:
            for v in VARIANTS:
                kl = v == "grpo"
                case = make_case(100 + len(names), T_seqs=8, G=4, V=37, max_len=4, mapping=mapping, kl=kl,
                                 stale=0.3)
                cfg = config(v, aggregation=agg, kl_weight=0.1 if kl else 0.0, engine_mismatch_cap=2.0)
                key = f"{mapping}_{agg}_{v}"
                names.append(key)
                if mapping == "B":
                    rows = case.row_of_token
                    ctx = np.arange(case.N, dtype=np.int32)
                    toffs = case.seq_offsets
                    adv_t = case.advantages
                    prox_tab = case.logits + np.random.default_rng(5).normal(0, 0.2, case.logits.shape)
                    lq = O.ref_log_probs(prox_tab, rows)[np.arange(case.T), case.token_ids]
                else:
                    rows = None
                    ctx = np.arange(case.T, dtype=np.int32)
                    toffs = np.arange(case.T + 1, dtype=np.int64)
                    adv_t = np.repeat(case.advantages, np.diff(case.seq_offsets))
                    lq = case.prox_logp
                    prox_tab = O.ref_build_prox_table(case.logits, case.token_ids, lq)
                val, grad = O.ref_loss_and_grad(cfg, case.logits, ctx, toffs, case.token_ids, adv_t,
                                                case.behavior_logp, prox_logits=prox_tab, ref_logits=case.ref_logits,
                                                engine_logp=case.engine_logp)
                lp = O.ref_log_probs(case.logits, np.arange(case.logits.shape[0], dtype=np.int32))
                out[key + "/logits"] = case.logits
                out[key + "/tokens"] = case.token_ids
                out[key + "/seq_offsets"] = toffs
                out[key + "/traj_context"] = ctx
                out[key + "/advantages"] = adv_t
                out[key + "/behavior"] = case.behavior_logp
                out[key + "/engine"] = case.engine_logp
                out[key + "/prox_logp"] = lq
                out[key + "/prox_table"] = prox_tab
                if case.ref_logits is not None:
                    out[key + "/ref_logits"] = case.ref_logits
                if rows is not None:
                    out[key + "/rows"] = rows
                out[key + "/value"] = np.array([val])
                out[key + "/grad"] = grad
                out[key + "/log_probs"] = lp
    out["loss_cases"] = np.array(names)

    # --- RngStream draws (rng.hpp:44-84) ---
    for kind, nm in [(0, "uniform"), (1, "normal"), (2, "u64")]:
        out[f"rng/{nm}"] = O.ref_rng_draws(42, "lengths", kind, 64)

    # --- toy_train_loop (bandit.cpp:41-119) ---
    tis = config("tis", aggregation="sequence_product", trunc_cap=5.0)
    r = O.ref_train_loop(tis, contexts=4, arms=10, group_size=8, traj_len=4, steps=300, lr=2.0, reward_noise=0.1,
                         async_lag=8, seed=1212)
    out["train/offpolicy_tis/final_reward"] = np.array([r["final_reward"]])
    out["train/offpolicy_tis/grad_norm_variance"] = np.array([r["grad_norm_variance"]])
    out["train/offpolicy_tis/reward"] = r["reward"]
    path = os.path.join(HERE, "golden_v1.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes;", len(names), "loss cases")


if __name__ == "__main__":
    main()
