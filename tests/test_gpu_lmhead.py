"""Experimental LM-head GEMM (tcgen05) with fused softmax statistics, against a
plain PyTorch fp32 reference of the same op (logits = H Wᵀ from the bf16 operands)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2510_11345_b200.lmhead import lmhead_dlogits, lmhead_lse  # noqa: E402


def _ref(H, W, tok):
    logits = H.float() @ W.float().t()
    return torch.logsumexp(logits.double(), dim=1), logits.gather(1, tok.long()[:, None])[:, 0].double()


@pytest.mark.parametrize("T,V,K", [(128, 256, 64), (300, 1000, 256), (256, 151936, 4096), (1, 517, 128)])
def test_lmhead_lse_matches_torch(T, V, K):
    g = torch.Generator(device="cuda")
    g.manual_seed(T * 7 + V + K)
    H = (torch.randn(T, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(V, K, device="cuda", generator=g) * (1.0 / K ** 0.5)).to(torch.bfloat16)
    tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    lse, xt = lmhead_lse(H, W, tok)
    torch.cuda.synchronize()
    rl, rx = _ref(H, W, tok)
    # fp32 accumulation in a different order + ex2.approx: absolute tolerance in log space
    assert torch.allclose(xt.double(), rx, atol=2e-3, rtol=1e-4), (xt - rx).abs().max()
    assert torch.allclose(lse.double(), rl, atol=2e-3, rtol=1e-5), (lse.double() - rl).abs().max()


@pytest.mark.parametrize("T,V,K", [(128, 256, 64), (300, 1003, 256), (256, 151936, 4096)])
def test_lmhead_dlogits_matches_torch(T, V, K):
    """The dlogits sweep: coef·(onehot − softmax) from recomputed logits, using the stats
    kernel's lse; against the fp32 torch reference, at the north-star dlogit tolerance."""
    g = torch.Generator(device="cuda")
    g.manual_seed(T + 3 * V + K)
    H = (torch.randn(T, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(V, K, device="cuda", generator=g) * (1.0 / K ** 0.5)).to(torch.bfloat16)
    tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    coef = torch.randn(T, device="cuda", generator=g, dtype=torch.float64) * 1e-3
    coef[::7] = 0.0
    lse, _ = lmhead_lse(H, W, tok)
    dl = lmhead_dlogits(H, W, tok, lse, coef)
    torch.cuda.synchronize()
    logits = (H.float() @ W.float().t()).double()
    p = torch.softmax(logits, dim=1)
    ref = -coef[:, None] * p
    ref[torch.arange(T, device="cuda"), tok.long()] += coef
    err = (dl.double() - ref).abs()
    bound = 2e-3 * coef.abs()[:, None] + 2.0 ** -8 * ref.abs() + 1e-30
    assert bool((err <= bound).all()), float((err / bound).max())


@pytest.mark.parametrize("variant", ["ppo", "tis", "decoupled_ppo", "cispo"])
def test_lmhead_loss_pipeline_matches_oracle(variant):
    """hidden states -> stats sweep -> per-token loss math -> dlogits sweep, against the fp64
    oracle run on the materialised logits H·Wᵀ.  The logits differ from the oracle's by the fp32
    accumulation order only, so values are compared at 1e-3 and clip decisions outside a 1e-3 band."""
    import numpy as np

    from paper_2510_11345_b200 import losses as L
    from paper_2510_11345_b200.lmhead import lmhead_loss_and_grad
    from tests.cases import config, make_case
    from tests.parity import run_oracle, to_device_batch

    case = make_case(31, T_seqs=8, G=4, V=1000, max_len=6, mapping="A", stale=0.2)
    T, V, K = case.T, case.V, 256
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    H = (torch.randn(T, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(V, K, device="cuda", generator=g) * (1.0 / K ** 0.5)).to(torch.bfloat16)
    logits = (H.float() @ W.float().t()).double()
    case.logits = logits.cpu().numpy()
    cfg = config(variant, engine_mismatch_cap=2.0)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    res = lmhead_loss_and_grad(cfg, H, W, pb)
    ref = run_oracle(case, cfg, normalization=1)
    g64 = lambda t: t.double().cpu().numpy()  # noqa: E731
    lp, ratio, coef = g64(res.token_logp), g64(res.token_ratio), g64(res.token_coef)
    assert np.allclose(lp, ref["token_logp"], atol=1e-3, rtol=0)
    assert np.allclose(ratio, ref["token_ratio"], rtol=2e-3, atol=0)
    r = ref["token_ratio"]
    band = np.zeros(T, dtype=bool)
    for edge in (1 - cfg.clip_eps, 1 + cfg.clip_eps, 1 - cfg.eps_low, 1 + cfg.eps_high, cfg.trunc_cap):
        band |= np.abs(r - edge) < 2e-3 * max(1.0, edge)
    ok = ~band
    assert np.allclose(coef[ok], ref["token_coef"][ok], rtol=2e-3, atol=1e-12)
    flags = res.token_flags.cpu().numpy()
    assert np.array_equal(flags[ok], ref["token_flags"][ok])
    D = g64(res.dlogits)
    R = ref["dlogits"]
    k = np.abs(ref["token_coef"])[:, None]
    err = np.abs(D - R)[ok]
    bound = (4e-3 * k + 2.0 ** -7 * np.abs(R))[ok] + 1e-30
    assert bool((err <= bound).all()), float((err / bound).max())
    val = float(res.scalars[0])
    assert abs(val - ref["value"]) <= 2e-3 * max(abs(ref["value"]), np.abs(ref["token_loss"]).sum() * 1e-3, 1e-30)
