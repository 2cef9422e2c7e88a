"""CPU: pin the oracle (oracle/rf_oracle.c) to the reference.

1. against the reference compiled from /root/reference (oracle/_ref), live, on
   random batches — every variant x aggregation x row mapping;
2. against the committed golden fixtures generated from the reference
   (tests/golden/golden_v1.npz, tests/golden/make_golden.py) — these travel to the
   GPU box, where /root/reference does not exist;
3. against the reference's own known-answer tests (proj/tests/test_offpolicy.cpp),
   restated here on the oracle.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2510_11345_b200.losses import LossConfig, LossVariant, RatioAggregation
from tests.cases import VARIANTS, config, make_case

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _oracle_on_golden(g, key):
    cfg_name = key.split("_", 2)
    mapping = key[0]
    agg = "sequence_product" if "_sequence_product_" in key else "token_mean"
    v = key.split("_" + agg + "_")[1]
    kl = v == "grpo"
    cfg = config(v, aggregation=agg, kl_weight=0.1 if kl else 0.0, engine_mismatch_cap=2.0)
    k = lambda n: g[key + "/" + n] if (key + "/" + n) in g.files else None
    rows = k("rows")
    res = O.oracle_loss_and_grad(cfg, k("logits"), k("tokens"), k("seq_offsets"), k("advantages"), k("behavior"),
                                 prox_logp=k("prox_logp"), engine_logp=k("engine"), row_of_token=rows,
                                 ref_logits=k("ref_logits"), normalization=0)
    C, V = k("logits").shape
    grad = np.zeros((C, V))
    if rows is None:
        grad = res["dlogits"]
    else:
        np.add.at(grad, rows, res["dlogits"])
    return cfg, res, grad


@pytest.mark.parametrize("key", list(np.load(GOLDEN)["loss_cases"]))
def test_oracle_matches_golden(key):
    g = np.load(GOLDEN)
    cfg, res, grad = _oracle_on_golden(g, key)
    assert res["status"] == 0
    ref_val = float(g[key + "/value"][0])
    assert abs(res["value"] - ref_val) <= 1e-13 * max(1.0, abs(ref_val))
    assert np.abs(grad - g[key + "/grad"]).max() <= 1e-15 + 1e-13 * np.abs(g[key + "/grad"]).max()
    # per-token log-probs equal ToyPolicy::log_probs at the sampled token
    lpt = g[key + "/log_probs"]
    rows = g[key + "/rows"] if key + "/rows" in g.files else np.arange(len(g[key + "/tokens"]))
    want = lpt[rows, g[key + "/tokens"]]
    assert np.abs(res["token_logp"] - want).max() <= 1e-14


def test_oracle_grpo_golden_bit_exact():
    g = np.load(GOLDEN)
    st, adv, deg = O.oracle_grpo(g["grpo_rewards"], g["grpo_offsets"])
    assert st == 0
    assert np.array_equal(adv, g["grpo_adv"])
    assert np.array_equal(deg, g["grpo_deg"])


@needs_ref
@pytest.mark.parametrize("mapping", ["A", "B"])
@pytest.mark.parametrize("agg", ["token_mean", "sequence_product"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_oracle_vs_live_reference(mapping, agg, variant):
    kl = variant == "grpo"
    case = make_case(7 + VARIANTS.index(variant), T_seqs=12, G=4, V=53, max_len=5, mapping=mapping, kl=kl,
                     stale=0.3)
    cfg = config(variant, aggregation=agg, kl_weight=0.1 if kl else 0.0, engine_mismatch_cap=2.0)
    if mapping == "B":
        rows = case.row_of_token
        prox_tab = case.logits + np.random.default_rng(5).normal(0, 0.2, case.logits.shape)
        lq = O.ref_log_probs(prox_tab, rows)[np.arange(case.T), case.token_ids]
        val, grad = O.ref_loss_and_grad(cfg, case.logits, np.arange(case.N, dtype=np.int32), case.seq_offsets,
                                        case.token_ids, case.advantages, case.behavior_logp, prox_logits=prox_tab,
                                        ref_logits=case.ref_logits, engine_logp=case.engine_logp)
        o = O.oracle_loss_and_grad(cfg, case.logits, case.token_ids, case.seq_offsets, case.advantages,
                                   case.behavior_logp, prox_logp=lq, engine_logp=case.engine_logp, row_of_token=rows,
                                   ref_logits=case.ref_logits)
        g2 = np.zeros_like(grad)
        np.add.at(g2, rows, o["dlogits"])
    else:
        T = case.T
        adv_t = np.repeat(case.advantages, np.diff(case.seq_offsets))
        offs = np.arange(T + 1, dtype=np.int64)
        prox_tab = O.ref_build_prox_table(case.logits, case.token_ids, case.prox_logp)
        val, grad = O.ref_loss_and_grad(cfg, case.logits, np.arange(T, dtype=np.int32), offs, case.token_ids,
                                        adv_t, case.behavior_logp, prox_logits=prox_tab, ref_logits=case.ref_logits,
                                        engine_logp=case.engine_logp)
        o = O.oracle_loss_and_grad(cfg, case.logits, case.token_ids, offs, adv_t, case.behavior_logp,
                                   prox_logp=case.prox_logp, engine_logp=case.engine_logp, ref_logits=case.ref_logits)
        g2 = o["dlogits"]
    assert o["status"] == 0
    assert abs(val - o["value"]) <= 1e-13 * max(1.0, abs(val))
    assert np.abs(grad - g2).max() <= 1e-13 * max(1.0, np.abs(grad).max())


@needs_ref
def test_oracle_grpo_vs_live_reference_and_throw():
    rng = np.random.default_rng(3)
    for _ in range(200):
        G = 2 + int(rng.integers(0, 14))
        r = rng.uniform(-3, 3, G)
        a, d = O.ref_grpo_advantages(r)
        st, a2, d2 = O.oracle_grpo(r, np.array([0, G]))
        assert st == 0 and np.array_equal(a, a2) and d == bool(d2[0])
    with pytest.raises(ValueError, match="group size must be >= 2"):
        O.ref_grpo_advantages(np.array([1.0]))
    assert O.oracle_grpo(np.array([1.0]), np.array([0, 1]))[0] == 13


# ---- the reference's known-answer tests (test_offpolicy.cpp), restated on the oracle ----
def _one_token(ratio, advantage, variant, **kw):
    """traj_with_ratio (test_offpolicy.cpp:16-23): ToyPolicy(1,4) all-zero logits."""
    logits = np.zeros((1, 4))
    lp = math.log(0.25)
    cfg = config(variant, **kw)
    return cfg, O.oracle_loss_and_grad(cfg, logits, np.array([0]), np.array([0, 1]), np.array([advantage]),
                                       np.array([lp - math.log(ratio)]), row_of_token=np.array([0]))


def test_grpo_hand_checked_groups():  # test_offpolicy.cpp:55-68
    assert list(O.oracle_grpo([1, 0, 1, 0], [0, 4])[1]) == [1, -1, 1, -1]
    assert list(O.oracle_grpo([2, 0], [0, 2])[1]) == [1, -1]
    st, a, d = O.oracle_grpo([0.5, 0.5, 0.5], [0, 3])
    assert d[0] == 1 and list(a) == [0, 0, 0]


def test_pinned_ratio_arithmetic():  # test_offpolicy.cpp:120-201
    lp = math.log(0.25)
    approx = lambda a, b: abs(a - b) <= 100 * 1.1920929e-07 * (1 + max(abs(a), abs(b)))
    assert approx(_one_token(1.5, 1.0, "ppo")[1]["value"], 1.2)
    assert approx(_one_token(0.5, -1.0, "ppo")[1]["value"], -0.8)
    assert approx(_one_token(10.0, 1.0, "tis", trunc_cap=5.0)[1]["value"], 5.0 * lp)
    assert approx(_one_token(0.5, 1.0, "tis", trunc_cap=5.0)[1]["value"], 0.5 * lp)
    assert approx(_one_token(1.5, 1.0, "cispo")[1]["value"], 1.2 * lp)
    assert approx(_one_token(0.7, 1.0, "cispo")[1]["value"], 0.8 * lp)
    assert approx(_one_token(3.0, 1.0, "topr", trunc_cap=1.0)[1]["value"], 1.0 * lp)
    assert approx(_one_token(3.0, -1.0, "topr", trunc_cap=1.0)[1]["value"], -1.0 * lp)
    assert approx(_one_token(0.4, -1.0, "topr", trunc_cap=1.0)[1]["value"], -0.4 * lp)
    assert approx(_one_token(3.0, 1.0, "topr", trunc_cap=1.0, w_plus=2.0, w_minus=0.5)[1]["value"], 2.0 * lp)
    assert approx(_one_token(0.4, -1.0, "topr", trunc_cap=1.0, w_plus=2.0, w_minus=0.5)[1]["value"],
                  -0.5 * 0.4 * lp)
    # flags: ppo clip zeroes the gradient (r=1.5, A=1), tis caps (r=10)
    assert _one_token(1.5, 1.0, "ppo")[1]["token_flags"][0] & 0x01
    assert _one_token(10.0, 1.0, "tis")[1]["token_flags"][0] & 0x01
    assert _one_token(3.0, 1.0, "topr", trunc_cap=1.0)[1]["token_flags"][0] & 0x02


def test_ppo_flat_beyond_clip():  # test_offpolicy.cpp:298-310
    for r in (1.3, 1.6, 2.4, 4.0):
        cfg, o = _one_token(r, 1.0, "ppo")
        assert abs(o["value"] - 1.2) < 1e-12
        assert np.all(o["dlogits"] == 0.0)  # clipped: gradient zeroed, row left at +0.0


def test_tis_inactive_cap_equals_naive_bit_exact():  # test_offpolicy.cpp:279-296
    case = make_case(7, T_seqs=8, G=4, V=5, max_len=2, mapping="B", stale=0.5)
    a = O.oracle_loss_and_grad(config("tis", trunc_cap=1e9), case.logits, case.token_ids, case.seq_offsets,
                               case.advantages, case.behavior_logp, row_of_token=case.row_of_token)
    b = O.oracle_loss_and_grad(config("naive_is"), case.logits, case.token_ids, case.seq_offsets, case.advantages,
                               case.behavior_logp, row_of_token=case.row_of_token)
    assert np.array_equal(a["dlogits"], b["dlogits"])


def test_ratio_one_reduces_to_reinforce():  # test_offpolicy.cpp:236-277, oracles.hpp:36-62
    case = make_case(6, T_seqs=8, G=4, V=5, max_len=2, mapping="B", stale=0.0, engine=False)
    from tests.cases import log_softmax_rows
    lp = log_softmax_rows(case.logits)
    beh = lp[case.row_of_token, case.token_ids]
    p = np.exp(lp)
    # independent REINFORCE gradient (oracle::reinforce_grad)
    want = np.zeros_like(case.logits)
    N = case.N
    for i in range(N):
        L = case.seq_offsets[i + 1] - case.seq_offsets[i]
        for t in range(case.seq_offsets[i], case.seq_offsets[i + 1]):
            w = case.advantages[i] / N / L
            ind = np.zeros(case.V)
            ind[case.token_ids[t]] = 1.0
            want[case.row_of_token[t]] += w * (ind - p[case.row_of_token[t]])
    for v in ["ppo", "tis", "cispo", "naive_is", "decoupled_ppo"]:
        o = O.oracle_loss_and_grad(config(v), case.logits, case.token_ids, case.seq_offsets, case.advantages, beh,
                                   prox_logp=beh, row_of_token=case.row_of_token)
        g = np.zeros_like(want)
        np.add.at(g, case.row_of_token, o["dlogits"])
        assert np.abs(g - want).max() < 1e-10, v


def test_error_codes_mirror_reference_throws():
    case = make_case(5, T_seqs=4, G=2, V=7, max_len=2, mapping="A")
    args = (case.logits, case.token_ids, case.seq_offsets, case.advantages, case.behavior_logp)
    assert O.oracle_loss_and_grad(config("decoupled_ppo"), *args)["status"] == 8   # missing prox
    assert O.oracle_loss_and_grad(config("grpo", kl_weight=0.5), *args)["status"] == 9  # missing ref
    assert O.oracle_loss_and_grad(config("tis", engine_mismatch_cap=3.0), *args)["status"] == 11
    assert O.oracle_loss_and_grad(config("ppo", clip_eps=1.5), *args)["status"] == 1
    assert O.oracle_loss_and_grad(config("tis", trunc_cap=0.0), *args)["status"] == 3
    bad = case.behavior_logp.copy()
    bad[0] = -1e6
    assert O.oracle_loss_and_grad(config("ppo"), case.logits, case.token_ids, case.seq_offsets, case.advantages,
                                  bad)["status"] == 12


@needs_ref
def test_reference_finite_differences_pass():  # test_offpolicy.cpp:312-338 (pins the _ref build)
    case = make_case(8, T_seqs=6, G=3, V=6, max_len=3, mapping="B", stale=0.3, scale=0.5)
    for v in ["ppo", "tis", "cispo", "topr"]:
        cfg = config(v)
        mre, checked, flagged = O.ref_finite_diff(cfg, case.logits, np.arange(case.N, dtype=np.int32),
                                                  case.seq_offsets, case.token_ids, case.advantages,
                                                  case.behavior_logp, h=1e-5)
        assert checked > 0 and mre < 1e-5, (v, mre)


def test_reference_train_loop_golden():
    """Acceptance criterion 12's TIS run (lag 8, sequence_product, seed 1212) from the golden file;
    live reference re-run when available."""
    g = np.load(GOLDEN)
    assert abs(float(g["train/offpolicy_tis/grad_norm_variance"][0]) - 0.01717) < 5e-5
    if O.ref_available():
        r = O.ref_train_loop(config("tis", aggregation="sequence_product"), contexts=4, arms=10, group_size=8,
                             traj_len=4, steps=300, lr=2.0, reward_noise=0.1, async_lag=8, seed=1212)
        assert r["final_reward"] == float(g["train/offpolicy_tis/final_reward"][0])


def test_sampled_row_checker_accepts_oracle_and_rejects_perturbations():
    """oracle/check.py (bench.py's --check leg): the oracle's own outputs pass, and a
    perturbed lp, a flipped flag, a coefficient taken from another row, or a dlogits row
    off by more than 2e-3·|k| are each rejected."""
    from oracle.check import check_sample
    from tests.cases import make_case

    case = make_case(61, T_seqs=12, G=4, V=257, max_len=5, mapping="A", stale=0.3)
    cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    kw = dict(logits=case.logits, token_ids=case.token_ids, seq_offsets=case.seq_offsets,
              advantages=case.advantages, behavior_logp=case.behavior_logp, prox_logp=case.prox_logp,
              engine_logp=case.engine_logp, ref_logits=None, normalization=1, global_num_seqs=case.N,
              global_num_tokens=case.T)
    ref = O.oracle_loss_and_grad(cfg, case.logits, case.token_ids, case.seq_offsets, case.advantages,
                                 case.behavior_logp, prox_logp=case.prox_logp, engine_logp=case.engine_logp,
                                 normalization=1)
    good = {"lp": ref["token_logp"].copy(), "ratio": ref["token_ratio"].copy(), "coef": ref["token_coef"].copy(),
            "loss": ref["token_loss"].copy(), "flags": ref["token_flags"].copy()}
    dl = {i: ref["dlogits"][i].copy() for i in range(0, case.T, 3)}
    assert check_sample(cfg, gpu=good, dl_rows=dl, **kw)["ok"]

    def bad(mut, rows=None):
        g = {k: v.copy() for k, v in good.items()}
        mut(g)
        return not check_sample(cfg, gpu=g, dl_rows=dl if rows is None else rows, **kw)["ok"]

    nz = int(np.nonzero(good["coef"])[0][0])
    assert bad(lambda g: g["lp"].__setitem__(0, g["lp"][0] * (1 + 1e-4)))
    assert bad(lambda g: g["flags"].__setitem__(1, g["flags"][1] ^ 0x01))
    assert bad(lambda g: g["coef"].__setitem__(nz, g["coef"][(nz + 1) % case.T] + 1e-9))
    rows = dict(dl)
    r0 = next(iter(rows))
    rows[r0] = rows[r0] + 3e-3 * max(abs(good["coef"][r0]), 1e-12)
    assert bad(lambda g: None, rows) or good["coef"][r0] == 0
