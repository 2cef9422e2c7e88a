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
