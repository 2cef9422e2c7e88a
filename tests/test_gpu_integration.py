"""GPU: the reference-side binding (integration/rlsim_gpu_shim.cpp).

The reference's own code — toy_train_loop (bandit.cpp:41-119) and the rest of
rlsim minus losses.cpp — is linked against rlsim's loss API implemented over the
C ABI (integration/Makefile -> integration/_build/librlsim_gpu.so).  These tests
drive that build through the same extern "C" driver as the CPU reference and
compare the two: loss_and_grad on the golden cases, and whole training runs.
"""
import os

import numpy as np
import pytest

import oracle as O
from tests.cases import config

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.gpu_shim_available(), reason="integration/_build/librlsim_gpu.so not built")]

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@pytest.mark.parametrize("key", [k for k in np.load(GOLDEN)["loss_cases"] if str(k).startswith("B_")])
def test_shim_loss_and_grad_matches_reference_golden(key):
    g = np.load(GOLDEN)
    agg = "sequence_product" if "_sequence_product_" in key else "token_mean"
    v = key.split("_" + agg + "_")[1]
    kl = v == "grpo"
    cfg = config(v, aggregation=agg, kl_weight=0.1 if kl else 0.0, engine_mismatch_cap=2.0)
    k = lambda n: g[key + "/" + n] if (key + "/" + n) in g.files else None
    val, grad = O.ref_loss_and_grad(cfg, k("logits"), k("traj_context"), k("seq_offsets"), k("tokens"),
                                    k("advantages"), k("behavior"), prox_logits=k("prox_table"),
                                    ref_logits=k("ref_logits"), engine_logp=k("engine"), lib=O.gpu_shim_lib())
    ref_val = float(k("value")[0])
    ref_grad = k("grad")
    scale = np.abs(ref_grad).max()
    assert abs(val - ref_val) <= 1e-5 * max(abs(ref_val), 1e-3 * np.abs(ref_grad).sum()), (val, ref_val)
    assert np.abs(grad - ref_grad).max() <= 1e-4 * scale + 1e-9, np.abs(grad - ref_grad).max() / scale


@pytest.mark.parametrize("variant,agg,lag,steps,lr,noise,seed,traj_len", [
    ("grpo", "token_mean", 0, 60, 0.8, 0.0, 12, 1),          # test_offpolicy.cpp:378-400
    ("tis", "token_mean", 4, 12, 0.5, 0.0, 3, 1),            # test_offpolicy.cpp:402-415
    ("tis", "sequence_product", 8, 300, 2.0, 0.1, 1212, 4),  # acceptance criterion 12 / offpolicy_tis.json
    ("decoupled_ppo", "token_mean", 2, 80, 0.5, 0.05, 7, 2),
    ("cispo", "token_mean", 3, 80, 0.5, 0.05, 9, 2),
])
def test_toy_train_loop_on_gpu_matches_reference(variant, agg, lag, steps, lr, noise, seed, traj_len):
    cfg = config(variant, aggregation=agg)
    kw = dict(contexts=4 if traj_len > 1 or seed == 1212 else 3, arms=10 if seed == 1212 else 6, group_size=8,
              traj_len=traj_len, steps=steps, lr=lr, reward_noise=noise, async_lag=lag, seed=seed)
    cpu = O.ref_train_loop(cfg, **kw)
    gpu = O.ref_train_loop(cfg, lib=O.gpu_shim_lib(), **kw)
    assert np.array_equal(cpu["staleness"], gpu["staleness"])
    # fp32 logits/dlogits on the GPU vs fp64 on the CPU: the learning curves agree closely
    assert np.abs(cpu["reward"] - gpu["reward"]).max() < 2e-3, np.abs(cpu["reward"] - gpu["reward"]).max()
    assert abs(cpu["final_reward"] - gpu["final_reward"]) < 1e-3 * cpu["final_reward"]
    assert gpu["final_reward"] > gpu["reward"][0] + 0.05 or steps < 50


@pytest.mark.parametrize("key", [k for k in np.load(GOLDEN)["loss_cases"] if str(k).startswith("B_")])
def test_python_policy_api_matches_reference_golden(key):
    """The rlsim-shaped Python API (losses.loss_and_grad_policy: Trajectory list + logits
    tables, grad folded per context on the device by rf_rows_segment_sum) on the same
    golden cases as the C++ shim."""
    import paper_2510_11345_b200 as rf

    g = np.load(GOLDEN)
    agg = "sequence_product" if "_sequence_product_" in key else "token_mean"
    v = key.split("_" + agg + "_")[1]
    kl = v == "grpo"
    cfg = config(v, aggregation=agg, kl_weight=0.1 if kl else 0.0, engine_mismatch_cap=2.0)
    k = lambda n: g[key + "/" + n] if (key + "/" + n) in g.files else None  # noqa: E731
    offs, ctx, tok, beh, eng = k("seq_offsets"), k("traj_context"), k("tokens"), k("behavior"), k("engine")
    batch = [rf.Trajectory(context=int(ctx[i]), tokens=tok[offs[i]:offs[i + 1]].tolist(),
                           advantage=float(k("advantages")[i]), behavior_logp=beh[offs[i]:offs[i + 1]].tolist(),
                           engine_logp=[] if eng is None else eng[offs[i]:offs[i + 1]].tolist())
             for i in range(len(ctx))]
    res = rf.loss_and_grad_policy(cfg, k("logits"), batch, prox_logits=k("prox_table"), ref_logits=k("ref_logits"))
    ref_val, ref_grad = float(k("value")[0]), k("grad").reshape(-1)
    grad = res.grad.numpy()
    scale = np.abs(ref_grad).max()
    assert abs(res.value - ref_val) <= 1e-5 * max(abs(ref_val), 1e-3 * np.abs(ref_grad).sum()), (res.value, ref_val)
    assert np.abs(grad - ref_grad).max() <= 1e-4 * scale + 1e-9, np.abs(grad - ref_grad).max() / scale
    again = rf.loss_and_grad_policy(cfg, k("logits"), batch, prox_logits=k("prox_table"), ref_logits=k("ref_logits"))
    assert np.array_equal(again.grad.numpy(), grad)  # deterministic fold
