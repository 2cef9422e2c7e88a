"""GPU: the LM-head fusion against the fp64 oracle at the
north-star tolerances.

The reference computes the loss from a logits row (ToyPolicy::log_probs,
policy.cpp:21-30, consumed at losses.cpp:159).  Here the logits are H·Wᵀ of bf16
hidden states and vocab projection, computed on the tensor cores with fp32
accumulation and never stored; the oracle runs on the EXACT fp64 logits of the same
bf16 operands (products of bf16 values are exact in fp64), so every difference is the
kernel's own fp32 accumulation and softmax arithmetic:

* lp / ratio / coefficient / token loss 1e-5 relative, flags bit-exact outside the
  kink band, dlogits |d − d_ref| ≤ 2e-3·|k| + half a bf16 ulp (tests/parity.py);
* the chunked backward dH = dlogits·W, dW = dlogitsᵀ·H against fp64 GEMMs of the
  oracle's dlogits, within the dlogit tolerance propagated through the GEMM.
"""
import numpy as np
import pytest
import torch

import oracle as O
from tests.cases import config, make_case
from tests.parity import DL_ABS, compare, run_oracle, to_device_batch

pytestmark = pytest.mark.gpu

from paper_2510_11345_b200 import losses as L  # noqa: E402
from paper_2510_11345_b200.lmhead import (lmhead_backward, lmhead_dlogits, lmhead_loss_and_grad,  # noqa: E402
                                          lmhead_lse)


def _operands(T, V, K, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    H = (torch.randn(T, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(V, K, device="cuda", generator=g) * (1.0 / K ** 0.5)).to(torch.bfloat16)
    return H, W, g


def _exact_logits(H, W):
    return H.double() @ W.double().t()  # exact products of bf16 values, fp64 sums


@pytest.mark.parametrize("T,V,K", [(128, 256, 64), (300, 1000, 256), (256, 151936, 4096), (1, 517, 128)])
def test_lmhead_lse_matches_oracle(T, V, K):
    H, W, g = _operands(T, V, K, T * 7 + V + K)
    tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    lse, xt = lmhead_lse(H, W, tok)
    torch.cuda.synchronize()
    X = _exact_logits(H, W).cpu().numpy()
    tk = tok.long().cpu().numpy()
    lp_ref = np.array([O.oracle_log_softmax(X[t])[tk[t]] for t in range(T)])
    lp = xt.double().cpu().numpy() - lse.cpu().numpy()
    rel = np.abs(lp - lp_ref) / np.maximum(np.abs(lp_ref), 1e-2)
    assert rel.max() <= 1e-5, rel.max()


@pytest.mark.parametrize("T,V,K", [(128, 256, 64), (300, 1003, 256), (256, 151936, 4096)])
def test_lmhead_dlogits_sweep_matches_fp64(T, V, K):
    """coef·(onehot − softmax) from recomputed logits and the stats sweep's lse."""
    H, W, g = _operands(T, V, K, T + 3 * V + K)
    tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    coef = torch.randn(T, device="cuda", generator=g, dtype=torch.float64) * 1e-3
    coef[::7] = 0.0
    lse, _ = lmhead_lse(H, W, tok)
    dl = lmhead_dlogits(H, W, tok, lse, coef)
    torch.cuda.synchronize()
    p = torch.softmax(_exact_logits(H, W), dim=1)
    ref = -coef[:, None] * p
    ref[torch.arange(T, device="cuda"), tok.long()] += coef
    err = (dl.double() - ref).abs()
    bound = DL_ABS * coef.abs()[:, None] + 2.0 ** -8 * ref.abs() + 1e-30
    assert bool((err <= bound).all()), float((err / bound).max())


@pytest.mark.parametrize("variant", ["ppo", "decoupled_ppo", "tis", "cispo", "topr", "naive_is"])
@pytest.mark.parametrize("V,K", [(1000, 256), (151936, 4096)])
def test_lmhead_loss_pipeline_matches_oracle(variant, V, K):
    """hidden states -> stats sweep -> per-token loss math -> dlogits sweep, against the fp64
    oracle on the exact logits, at the north-star tolerances (tests/parity.compare)."""
    case = make_case(31, T_seqs=8, G=4, V=8, max_len=8, mapping="A", stale=0.2)
    T = case.T
    H, W, g = _operands(T, V, K, 5 + V)
    X = _exact_logits(H, W)
    case.logits = X.cpu().numpy()
    # tokens from the real softmax, log-probs of the behaviour/prox/engine policies around it
    rng = np.random.default_rng(9)
    lp_all = X - torch.logsumexp(X, dim=1, keepdim=True)
    case.token_ids = torch.multinomial(lp_all.exp(), 1, generator=g).squeeze(1).int().cpu().numpy()
    lp = lp_all.gather(1, torch.from_numpy(case.token_ids).long().cuda()[:, None])[:, 0].cpu().numpy()
    delta = rng.normal(0, 0.2, T)
    case.behavior_logp, case.prox_logp = lp - delta, lp - delta / 2
    case.engine_logp = case.behavior_logp - rng.normal(0, 0.01, T)
    cfg = config(variant, engine_mismatch_cap=2.0)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    res = lmhead_loss_and_grad(cfg, H, W, pb)
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, res, ref)


@pytest.mark.parametrize("chunk", [16384, 4096])
def test_lmhead_backward_matches_fp64(chunk):
    """dH = dlogits·W and dW = dlogitsᵀ·H from vocabulary chunks (the last chunk partial),
    against fp64 GEMMs of the exact-logit dlogits.  Bound: the north-star dlogit tolerance
    propagated through the GEMM, Σ_v (2e-3·|k| + 2^-8·|R_v|)·|W_v| (and ·|H| for dW)."""
    T, V, K = 192, 151936 if chunk == 16384 else 40000, 1024
    H, W, g = _operands(T, V, K, 77 + chunk)
    tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    coef = torch.randn(T, device="cuda", generator=g, dtype=torch.float64) * 1e-3
    lse, _ = lmhead_lse(H, W, tok)
    dH, dW = lmhead_backward(H, W, tok, lse, coef, chunk_vocab=chunk)
    torch.cuda.synchronize()
    p = torch.softmax(_exact_logits(H, W), dim=1)
    R = -coef[:, None] * p
    R[torch.arange(T, device="cuda"), tok.long()] += coef
    W64, H64 = W.double(), H.double()
    per = DL_ABS * coef.abs()[:, None] + 2.0 ** -8 * R.abs()  # per-element dlogit tolerance
    dH_ref, dW_ref = R @ W64, R.t() @ H64
    bH = per @ W64.abs() + 1e-6 * (R.abs() @ W64.abs()) + 1e-30
    bW = per.t() @ H64.abs() + 1e-6 * (R.abs().t() @ H64.abs()) + 1e-30
    eH, eW = (dH.double() - dH_ref).abs(), (dW.double() - dW_ref).abs()
    assert bool((eH <= bH).all()), float((eH / bH).max())
    assert bool((eW <= bW).all()), float((eW / bW).max())


def test_lmhead_loss_and_grads_pipeline():
    """want="grads": the loss scalars and per-token outputs match the dlogits pipeline, and
    (dH, dW) equal the GEMMs of that pipeline's dlogits."""
    case = make_case(33, T_seqs=8, G=4, V=8, max_len=8, mapping="A", stale=0.2)
    T, V, K = case.T, 20000, 512
    H, W, g = _operands(T, V, K, 99)
    X = _exact_logits(H, W)
    case.token_ids = torch.multinomial(torch.softmax(X, 1), 1, generator=g).squeeze(1).int().cpu().numpy()
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    pb.logits = torch.empty(1, V, dtype=torch.bfloat16, device="cuda")  # placeholder: never read
    pb.vocab = V
    cfg = config("tis")
    a = lmhead_loss_and_grad(cfg, H, W, pb)
    b, dH, dW = lmhead_loss_and_grad(cfg, H, W, pb, want="grads", chunk_vocab=4096)
    for n in ("token_logp", "token_ratio", "token_coef", "token_loss", "token_flags", "scalars"):
        assert torch.equal(getattr(a, n), getattr(b, n)), n
    assert b.dlogits is None
    dl = a.dlogits.float()
    assert torch.allclose(dH, dl @ W.float(), rtol=1e-3, atol=1e-7)
    assert torch.allclose(dW, dl.t() @ H.float(), rtol=1e-3, atol=1e-7)
