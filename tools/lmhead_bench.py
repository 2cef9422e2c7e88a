"""Throughput of the experimental LM-head GEMM + fused softmax statistics
(rf_lmhead_lse) against cuBLAS bf16 GEMM of the same shape (logits materialised)
followed by torch's logsumexp (run on the GPU box):
    python tools/lmhead_bench.py [--tokens 8192] [--vocab 151936] [--hidden 4096]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_11345_b200.lmhead import lmhead_dlogits, lmhead_lse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=8192)
ap.add_argument("--vocab", type=int, default=151936)
ap.add_argument("--hidden", type=int, default=4096)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
T, V, K = a.tokens, a.vocab, a.hidden
g = torch.Generator(device="cuda")
g.manual_seed(0)
H = (torch.randn(T, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
W = (torch.randn(V, K, device="cuda", generator=g) * (1.0 / K ** 0.5)).to(torch.bfloat16)
tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
flops = 2.0 * T * V * K


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


ms_fused = timed(lambda: lmhead_lse(H, W, tok))


def unfused():
    logits = H @ W.t()
    return torch.logsumexp(logits.float(), dim=1)


lse0, _ = lmhead_lse(H, W, tok)
coef = torch.full((T,), 1e-4, dtype=torch.float64, device="cuda")
ms_dl = timed(lambda: lmhead_dlogits(H, W, tok, lse0, coef))


def unfused_dl():
    logits = H @ W.t()
    p = torch.softmax(logits.float(), dim=1)
    d = (-coef[:, None].float() * p)
    d[torch.arange(T, device="cuda"), tok.long()] += coef.float()
    return d.to(torch.bfloat16)


ms_gemm = timed(lambda: H @ W.t())
ms_unfused_dl = timed(unfused_dl) if T * V <= 8192 * 151936 else None
ms_unfused = timed(unfused)
# End-to-end loss + dlogits from hidden states: the fused pipeline (two tensor-core sweeps,
# no logits tensor) against cuBLAS logits (materialised, bf16) + the fused ring loss kernel.
import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402
from paper_2510_11345_b200.lmhead import lmhead_loss_and_grad  # noqa: E402

L_seq = 8
nseq = T // L_seq
seq_offsets = torch.arange(0, nseq + 1, device="cuda", dtype=torch.int64) * L_seq
lse_r, xt_r = lmhead_lse(H, W, tok)
lp0 = (xt_r - lse_r).double()
behavior = (lp0 - 0.05 * torch.randn(T, device="cuda", generator=g, dtype=torch.float64)).float()
adv = torch.randn(nseq, device="cuda", generator=g, dtype=torch.float64)
logits_buf = torch.empty(T, (V + 7) // 8 * 8, dtype=torch.bfloat16, device="cuda")[:, :V]
pb = L.PackedBatch(logits=logits_buf, token_ids=tok, seq_offsets=seq_offsets, advantages=adv, behavior_logp=behavior,
                   normalization=L.Normalization.global_token)
cfg = L.LossConfig()  # PPO-clip
op = rf.OffPolicyLoss(cfg, pb, chunk_tokens=T)


def composed():
    torch.matmul(H, W.t(), out=logits_buf)
    op.zero()
    op.run(pb, 0, T)


ms_composed = timed(composed)
ms_pipeline = timed(lambda: lmhead_loss_and_grad(cfg, H, W, pb, check=False))


def composed_grads():  # + the backward GEMMs of the materialised dlogits (cuBLAS, fp32 out)
    composed()
    dl = op.dlogits
    return torch.mm(dl, W, out_dtype=torch.float32), torch.mm(dl.t(), H, out_dtype=torch.float32)


ms_composed_grads = timed(composed_grads)
ms_pipeline_grads = timed(lambda: lmhead_loss_and_grad(cfg, H, W, pb, check=False, want="grads"))
grads_by_chunk = {c: round(timed(lambda: lmhead_loss_and_grad(cfg, H, W, pb, check=False, want="grads",
                                                               chunk_vocab=c)), 3)
                  for c in (8192, 16384, 24576, 32768)}
def peak_gb(fn):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    fn()
    torch.cuda.synchronize()
    return round((torch.cuda.max_memory_allocated() - base) / 1e9, 2)


peak_fused = peak_gb(lambda: lmhead_loss_and_grad(cfg, H, W, pb, check=False, want="grads"))
peak_composed = peak_gb(composed_grads)  # logits_buf and op.dlogits are preallocated: add them below
ms_bwd_gemms = timed(lambda: (torch.mm(op.dlogits, W, out_dtype=torch.float32),
                              torch.mm(op.dlogits.t(), H, out_dtype=torch.float32)))
peaks = {}
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
        peaks = json.load(f)
except Exception:
    pass
peak = float(peaks.get("bf16_tflops", peaks.get("dense_bf16_tflops", 0)) or 0)
out = {"tokens": T, "vocab": V, "hidden": K, "fused_ms": round(ms_fused, 3),
       "fused_tflops": round(flops / ms_fused / 1e9, 1), "cublas_gemm_ms": round(ms_gemm, 3),
       "cublas_gemm_tflops": round(flops / ms_gemm / 1e9, 1), "cublas_gemm_plus_logsumexp_ms": round(ms_unfused, 3),
       "logits_bytes_avoided": T * V * 2 * 2, "measured_bf16_peak_tflops": peak or None,
       "fused_dlogits_ms": round(ms_dl, 3), "fused_dlogits_tflops": round(flops / ms_dl / 1e9, 1),
       "fused_stats_plus_dlogits_ms": round(ms_fused + ms_dl, 3),
       "cublas_gemm_plus_torch_softmax_dlogits_ms": None if ms_unfused_dl is None else round(ms_unfused_dl, 3),
       "loss_and_dlogits_fused_pipeline_ms": round(ms_pipeline, 3),
       "loss_and_dlogits_cublas_logits_plus_ring_kernel_ms": round(ms_composed, 3),
       "loss_and_grads_fused_pipeline_ms": round(ms_pipeline_grads, 3),
       "loss_and_grads_fused_ms_by_chunk_vocab": grads_by_chunk,
       "loss_and_grads_composed_ms": round(ms_composed_grads, 3),
       "backward_gemms_cublas_ms": round(ms_bwd_gemms, 3),
       "peak_extra_GB_fused_grads": peak_fused,
       "peak_extra_GB_composed_grads": round(peak_composed + 2 * T * V * 2 / 1e9, 2)}
print(json.dumps(out))
