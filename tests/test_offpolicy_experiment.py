"""The reference's `offpolicy` experiment mode end to end (configs/offpolicy_tis.json
-> experiment.cpp:589-622 -> toy_train_loop, bandit.cpp:41-119 -> loss_and_grad).

* CPU: oracle/_ref/rlsim_simulate_ref (the unmodified reference library) reproduces
  the committed golden rows exactly (pins the harness and the fixture);
* GPU: integration/_build/rlsim_simulate_gpu — the same unmodified experiment code
  with every loss_and_grad / grpo_advantages / trajectory_ratio call going through
  integration/rlsim_gpu_shim.cpp and the C ABI — reproduces them within the
  training-loop tolerance (fp32 logits and dlogits on the GPU vs fp64 on the CPU,
  accumulated over 300 optimiser steps).
"""
import json
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "offpolicy_golden.json")
REF_SIM = os.path.join(ROOT, "oracle", "_ref", "rlsim_simulate_ref")
GPU_SIM = os.path.join(ROOT, "integration", "_build", "rlsim_simulate_gpu")

CASES = json.load(open(GOLDEN))["cases"]


def simulate(binary, cfg):
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(cfg, f)
        path = f.name
    try:
        r = subprocess.run([binary, path], capture_output=True, text=True, timeout=900)
    finally:
        os.unlink(path)
    assert r.returncode == 0, r.stderr
    rows = [json.loads(x) for x in r.stdout.splitlines()]
    assert not any(x["metric"] == "error" for x in rows), rows
    return {x["metric"]: x["value"] for x in rows if x["rep"] == 0}


@pytest.mark.skipif(not os.path.exists(REF_SIM), reason="oracle/_ref/rlsim_simulate_ref not built")
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_reference_simulate_reproduces_golden(case):
    assert simulate(REF_SIM, case["config"]) == case["reference"]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(GPU_SIM), reason="integration/_build/rlsim_simulate_gpu not built")
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_gpu_simulate_matches_reference(case):
    got = simulate(GPU_SIM, case["config"])
    ref = case["reference"]
    assert got["steps"] == ref["steps"]
    # final expected reward of the learned policy after 300 steps: 2e-3 absolute
    assert abs(got["final_reward"] - ref["final_reward"]) <= 2e-3, (got, ref)
    # the variance of the per-step gradient norms: 5% relative
    assert abs(got["grad_norm_variance"] - ref["grad_norm_variance"]) <= 0.05 * ref["grad_norm_variance"], (got, ref)
