"""Experimental: the LM-head GEMM with the softmax statistics fused into its
epilogue ("fusion with the step before").

``lmhead_lse(hidden, w_vocab, token_ids)`` returns ``lse[t] = logsumexp_v (H Wᵀ)[t, v]``
and ``x_tok[t] = (H Wᵀ)[t, token_ids[t]]`` computed by ``rf_lmhead_lse``
(``csrc/rf_lmhead.cu``: TMA + tcgen05.mma into tensor memory, fp32 accumulation,
online max/Σexp in the epilogue) without materialising the [T, V] logits.  From
these, ``lp = x_tok - lse`` is the per-token log-prob the loss needs."""
from __future__ import annotations

import torch

from . import _abi


def lmhead_lse(hidden: torch.Tensor, w_vocab: torch.Tensor, token_ids: torch.Tensor, stream=None):
    if hidden.dtype != torch.bfloat16 or w_vocab.dtype != torch.bfloat16:
        raise TypeError("hidden and w_vocab must be bf16")
    if hidden.dim() != 2 or w_vocab.dim() != 2 or hidden.shape[1] != w_vocab.shape[1]:
        raise ValueError("hidden [T, K] and w_vocab [V, K] expected")
    if not (hidden.is_contiguous() and w_vocab.is_contiguous()):
        raise ValueError("row-major contiguous operands expected")
    T, K = hidden.shape
    V = w_vocab.shape[0]
    tok = token_ids.to(device=hidden.device, dtype=torch.int32).contiguous()
    lse = torch.empty(T, dtype=torch.float32, device=hidden.device)
    xt = torch.empty(T, dtype=torch.float32, device=hidden.device)
    lib = _abi.load_library()
    s = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    st = lib.rf_lmhead_lse(hidden.data_ptr(), w_vocab.data_ptr(), tok.data_ptr(), T, V, K, lse.data_ptr(),
                           xt.data_ptr(), s)
    if st != 0:
        from .losses import status_string

        raise RuntimeError(f"rf_lmhead_lse: {status_string(st)}")
    return lse, xt


def lmhead_dlogits(hidden: torch.Tensor, w_vocab: torch.Tensor, token_ids: torch.Tensor, lse: torch.Tensor,
                   coef: torch.Tensor, stream=None) -> torch.Tensor:
    """dlogits[t, v] = coef[t]·(1[v = tok_t] − exp((H Wᵀ)[t, v] − lse[t])), bf16, from a second
    tensor-core sweep (the logits are recomputed, never stored)."""
    T, K = hidden.shape
    V = w_vocab.shape[0]
    padV = (V + 7) // 8 * 8
    out = torch.empty(T, padV, dtype=torch.bfloat16, device=hidden.device)
    tok = token_ids.to(device=hidden.device, dtype=torch.int32).contiguous()
    lse32 = lse.to(torch.float32).contiguous()
    c64 = coef.to(torch.float64).contiguous()
    lib = _abi.load_library()
    s = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    st = lib.rf_lmhead_dlogits(hidden.data_ptr(), w_vocab.data_ptr(), tok.data_ptr(), T, V, K, lse32.data_ptr(),
                               c64.data_ptr(), out.data_ptr(), padV, s)
    if st != 0:
        from .losses import status_string

        raise RuntimeError(f"rf_lmhead_dlogits: {status_string(st)}")
    return out[:, :V]
