"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Mirrors the reference's own test strategy (proj/tests/test_offpolicy.cpp):
every variant, both aggregations, both kernels, both row mappings, bf16 and
f32 logits, ragged/odd vocabularies, plus size-independent properties at the
full Qwen3 vocabulary.
"""
import numpy as np
import pytest
import torch

from tests.cases import VARIANTS, config, make_case
from tests.parity import compare, run_oracle, to_device_batch

pytestmark = pytest.mark.gpu

import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402

TOKEN_MEAN_VARIANTS = ["ppo", "decoupled_ppo", "tis", "cispo", "topr", "grpo", "naive_is"]


def _cfg(v, **kw):
    return config(v, engine_mismatch_cap=kw.pop("cap", 2.0), **kw)


@pytest.mark.parametrize("variant", TOKEN_MEAN_VARIANTS)
@pytest.mark.parametrize("kernel", ["ring", "generic"])
def test_token_mean_v32k_mapping_a(variant, kernel):
    case = make_case(11, T_seqs=16, G=8, V=32000, max_len=24, mapping="A", stale=0.2, alpha=2)
    cfg = _cfg(variant)
    norm = L.Normalization.global_token
    pb = to_device_batch(case, normalization=norm)
    gpu = rf.loss_and_grad(cfg, pb, kernel=kernel)
    ref = run_oracle(case, cfg, normalization=int(norm))
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("variant", ["ppo", "decoupled_ppo", "tis", "topr", "cispo"])
def test_token_mean_qwen3_vocab_cluster(variant):
    """V = 151,936: the row spans a 2-CTA cluster (DSMEM softmax exchange)."""
    case = make_case(12, T_seqs=8, G=4, V=151936, max_len=10, mapping="A", stale=0.3, alpha=8)
    cfg = _cfg(variant)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("V", [2, 6, 1003, 4099, 32000 + 5])
@pytest.mark.parametrize("kernel", ["auto", "generic"])
def test_odd_vocab(V, kernel):
    case = make_case(13, T_seqs=6, G=3, V=V, max_len=6, mapping="A", stale=0.2)
    cfg = _cfg("tis")
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel=kernel)
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("variant", ["ppo", "tis", "decoupled_ppo"])
@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
def test_f32_logits(variant, out):
    case = make_case(14, T_seqs=8, G=4, V=32000, max_len=8, mapping="A", round_bf16=False, stale=0.2)
    case.logits = case.logits.astype(np.float32).astype(np.float64)
    cfg = _cfg(variant)
    pb = to_device_batch(case, dtype=torch.float32, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, dlogits_dtype=out, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref, out_dtype=out)


def test_f32_logits_qwen3_vocab_cluster4():
    """f32 rows of 151,936 (608 KB) span a 4-CTA cluster."""
    case = make_case(15, T_seqs=4, G=2, V=151936, max_len=4, mapping="A", round_bf16=False, stale=0.2)
    case.logits = case.logits.astype(np.float32).astype(np.float64)
    cfg = _cfg("cispo")
    pb = to_device_batch(case, dtype=torch.float32, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, dlogits_dtype=torch.float32, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref, out_dtype=torch.float32)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("kernel", ["auto", "generic"])
def test_mapping_b_reference_normalisation(variant, kernel):
    """Rows shared per sequence, 1/(N*L_i) normalisation (reference layout)."""
    kl = variant == "grpo"
    case = make_case(16, T_seqs=12, G=4, V=4096, max_len=9, mapping="B", stale=0.3, kl=kl)
    cfg = _cfg(variant, kl_weight=0.1 if kl else 0.0)
    pb = to_device_batch(case, with_ref=kl)
    gpu = rf.loss_and_grad(cfg, pb, kernel=kernel)
    ref = run_oracle(case, cfg, normalization=0)
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("variant", VARIANTS)
def test_sequence_product(variant):
    kl = variant == "grpo"
    case = make_case(17, T_seqs=12, G=4, V=4096, max_len=7, mapping="A", stale=0.05, kl=kl)
    cfg = _cfg(variant, aggregation="sequence_product", kl_weight=0.1 if kl else 0.0)
    pb = to_device_batch(case, with_ref=kl)
    gpu = rf.loss_and_grad(cfg, pb)
    ref = run_oracle(case, cfg, normalization=0)
    compare(case, cfg, gpu, ref)


def test_grpo_kl_token_mean_mapping_a():
    case = make_case(18, T_seqs=8, G=4, V=32000, max_len=6, mapping="A", stale=0.2, kl=True)
    cfg = _cfg("grpo", kl_weight=0.1)
    pb = to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb)
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("V", [1003, 4099, 32000, 151936])
@pytest.mark.parametrize("kernel", ["ring", "generic"])
def test_grpo_kl_fast_path(V, kernel):
    """Exact-KL GRPO on the lag kernel (policy + reference rows co-resident; the
    Qwen3 row spans a 4-CTA cluster) against the oracle, and the generic kernel."""
    case = make_case(21, T_seqs=6 if V > 100000 else 12, G=3, V=V, max_len=6, mapping="A", stale=0.2, kl=True)
    cfg = _cfg("grpo", kl_weight=0.1)
    pb = to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel=kernel)
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
def test_grpo_kl_fast_path_mapping_b(out):
    """Rows shared per sequence (KL per trajectory through the 1/(N·L_i) scale)."""
    case = make_case(22, T_seqs=12, G=4, V=32000, max_len=9, mapping="B", stale=0.3, kl=True)
    cfg = _cfg("grpo", kl_weight=0.25)
    pb = to_device_batch(case, with_ref=True)
    gpu = rf.loss_and_grad(cfg, pb, dlogits_dtype=out, kernel="ring")
    ref = run_oracle(case, cfg, normalization=0)
    compare(case, cfg, gpu, ref, out_dtype=out)


def test_f32_logp_inputs_and_grad_sign():
    case = make_case(19, T_seqs=8, G=4, V=32000, max_len=8, mapping="A", stale=0.2)
    cfg = _cfg("ppo")
    pb = to_device_batch(case, logp_dtype=torch.float32, grad_sign=-1.0, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb)
    ref = run_oracle(case, cfg, normalization=1, logp_dtype=torch.float32, grad_sign=-1.0)
    compare(case, cfg, gpu, ref, logp_dtype=torch.float32)


def test_grpo_advantages_bit_exact():
    import oracle as O

    rng = np.random.default_rng(3)
    sizes = rng.integers(2, 31, 500)
    go = np.zeros(len(sizes) + 1, dtype=np.int64)
    go[1:] = np.cumsum(sizes)
    rewards = rng.uniform(-5, 5, go[-1])
    # every 5th group flat -> degenerate
    for g in range(0, len(sizes), 5):
        rewards[go[g]:go[g + 1]] = rewards[go[g]]
    adv, deg = rf.grpo_advantages(torch.from_numpy(rewards).cuda(), torch.from_numpy(go).cuda())
    st, adv_o, deg_o = O.oracle_grpo(rewards, go)
    assert st == 0
    assert np.array_equal(adv.cpu().numpy(), adv_o)
    assert np.array_equal(deg.cpu().numpy(), deg_o)
    if O.ref_available():
        for g in range(len(sizes)):
            a, d = O.ref_grpo_advantages(rewards[go[g]:go[g + 1]])
            assert np.array_equal(a, adv_o[go[g]:go[g + 1]]) and d == bool(deg_o[g])


def test_streaming_chunks_equal_single_call():
    """Chunked calls (accumulating scalars) == one call: per-token outputs bit-equal."""
    case = make_case(20, T_seqs=16, G=8, V=32000, max_len=20, mapping="A", stale=0.2)
    cfg = _cfg("decoupled_ppo")
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    one = rf.loss_and_grad(cfg, pb)
    op = rf.OffPolicyLoss(cfg, pb, chunk_tokens=37)
    op.zero()
    dl = []
    for t0 in range(0, pb.num_tokens, 37):
        t1 = min(pb.num_tokens, t0 + 37)
        op.run(pb, t0, t1)
        dl.append(op.dlogits[: t1 - t0].clone())
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(dl), one.dlogits)
    for name in ["token_logp", "token_ratio", "token_coef", "token_loss", "token_flags"]:
        assert torch.equal(getattr(op, name), getattr(one, name)), name
    assert abs(float(op.scalars[0]) - one.value) <= 1e-12 * max(1.0, abs(one.value))


def test_deterministic_rerun():
    case = make_case(21, T_seqs=8, G=4, V=151936, max_len=6, mapping="A", stale=0.2)
    cfg = _cfg("tis")
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    a = rf.loss_and_grad(cfg, pb)
    b = rf.loss_and_grad(cfg, pb)
    assert torch.equal(a.dlogits, b.dlogits)
    assert torch.equal(a.scalars, b.scalars)


def test_dlogit_rows_sum_to_zero_full_vocab():
    """Size-independent property: sum_v k (onehot - p_v) = 0 for every row."""
    case = make_case(22, T_seqs=16, G=8, V=151936, max_len=64, mapping="A", stale=0.2)
    cfg = _cfg("cispo")
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, dlogits_dtype=torch.float32)
    rs = gpu.dlogits.double().sum(dim=1).abs()
    k = gpu.token_coef.abs()
    assert bool((rs <= 1e-3 * k + 1e-30).all()), float((rs / k.clamp_min(1e-300)).max())


def test_nonfinite_ratio_raises():
    case = make_case(23, T_seqs=4, G=2, V=1024, max_len=3, mapping="A")
    case.behavior_logp[1] = -1e6  # exp(lp - b) overflows
    cfg = _cfg("ppo")
    pb = to_device_batch(case)
    with pytest.raises(rf.InvalidArgument, match="non-finite ratio"):
        rf.loss_and_grad(cfg, pb)


def test_missing_inputs_raise():
    case = make_case(24, T_seqs=4, G=2, V=1024, max_len=3, mapping="A")
    pb = to_device_batch(case)
    pb.prox_logp = None
    with pytest.raises(rf.InvalidArgument, match="proximal"):
        rf.loss_and_grad(_cfg("decoupled_ppo"), pb)
    with pytest.raises(rf.InvalidArgument, match="reference policy"):
        rf.loss_and_grad(_cfg("grpo", kl_weight=0.5), pb)
    pb.engine_logp = None
    with pytest.raises(rf.InvalidArgument, match="engine"):
        rf.loss_and_grad(_cfg("tis", cap=5.0), pb)


@pytest.mark.parametrize("variant", ["ppo", "tis", "topr", "cispo", "decoupled_ppo", "naive_is"])
@pytest.mark.parametrize("V", [32000, 151936])
def test_sequence_product_fast_path(variant, V):
    """Ring stats pass + sequence scalars + streaming dlogits pass (ring-compatible layout)."""
    case = make_case(25, T_seqs=8, G=4, V=V, max_len=6, mapping="A", stale=0.05)
    cfg = _cfg(variant, aggregation="sequence_product")
    pb = to_device_batch(case, normalization=L.Normalization.seq_then_batch)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=0)
    compare(case, cfg, gpu, ref)
    gen = rf.loss_and_grad(cfg, pb, kernel="generic")
    assert torch.equal(gpu.token_flags, gen.token_flags)


def test_sequence_product_mapping_b_fast_path():
    case = make_case(26, T_seqs=12, G=4, V=32000, max_len=9, mapping="B", stale=0.1)
    cfg = _cfg("tis", aggregation="sequence_product")
    pb = to_device_batch(case)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=0)
    compare(case, cfg, gpu, ref)


@pytest.mark.parametrize("V,f32", [(4099, False), (32005, True), (151936, False)])
def test_sequence_product_long_sequences(V, f32):
    """Sequences spanning many 32-token blocks (K2s prefetch + sequential sums), odd
    vocabulary tails and f32 logits through the streaming stats pass (K2st)."""
    case = make_case(27, T_seqs=8, G=4, V=V, max_len=160, mapping="A", round_bf16=not f32, stale=0.01)
    assert np.diff(case.seq_offsets).max() > 64
    dt = torch.float32 if f32 else torch.bfloat16
    if f32:
        case.logits = case.logits.astype(np.float32).astype(np.float64)
    for variant in ["tis", "decoupled_ppo"]:
        cfg = _cfg(variant, aggregation="sequence_product")
        pb = to_device_batch(case, dtype=dt, normalization=L.Normalization.seq_then_batch)
        gpu = rf.loss_and_grad(cfg, pb, dlogits_dtype=dt, kernel="ring")
        ref = run_oracle(case, cfg, normalization=0)
        compare(case, cfg, gpu, ref, out_dtype=dt)


def test_grpo_kl_groups_many_rows():
    """Exact KL at Qwen3 vocab with several rows per CTA group (the L2 exchange slots
    wrap, row % 4) and two launches (a new epoch in the sequence words): parity, and
    the second launch bit-identical to the first."""
    case = make_case(28, T_seqs=20, G=4, V=151936, max_len=64, mapping="A", stale=0.2, kl=True)
    assert case.T > 4 * 37
    cfg = _cfg("grpo", kl_weight=0.1)
    pb = to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel="ring")
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)
    again = rf.loss_and_grad(cfg, pb, kernel="ring")
    assert torch.equal(gpu.dlogits, again.dlogits)
    assert torch.equal(gpu.scalars, again.scalars)


_AB_ARM = r"""
import sys
sys.path.insert(0, {root!r})
import paper_2510_11345_b200 as rf
from paper_2510_11345_b200 import losses as L
from tests.cases import config, make_case
from tests.parity import compare, run_oracle, to_device_batch
kl = {kl!r}
case = make_case(29, T_seqs=8, G=4, V=151936, max_len=40, mapping="A", stale=0.1, kl=kl)
if kl:
    cfg = config("grpo", engine_mismatch_cap=2.0, kl_weight=0.1)
    pb = to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    ref = run_oracle(case, cfg, normalization=1)
else:
    cfg = config("tis", engine_mismatch_cap=2.0, aggregation="sequence_product")
    pb = to_device_batch(case, normalization=L.Normalization.seq_then_batch)
    ref = run_oracle(case, cfg, normalization=0)
compare(case, cfg, rf.loss_and_grad(cfg, pb, kernel="ring"), ref)
print("arm ok")
"""


@pytest.mark.parametrize("env,kl", [({"RF_KL_GX": "0"}, True)])
def test_ab_arms_parity(env, kl):
    """The exact-KL hardware-cluster kernel (the fallback when the cooperative CTA-group
    launch cannot place every CTA; selected with RF_KL_GX=0, read once per process, so
    it runs in a subprocess)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _AB_ARM.format(root=root, kl=kl)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "arm ok" in r.stdout, r.stdout + r.stderr
