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
    lse = torch.empty(T, dtype=torch.float64, device=hidden.device)
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
    lse64 = lse.to(torch.float64).contiguous()
    c64 = coef.to(torch.float64).contiguous()
    lib = _abi.load_library()
    s = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    st = lib.rf_lmhead_dlogits(hidden.data_ptr(), w_vocab.data_ptr(), tok.data_ptr(), T, V, K, lse64.data_ptr(),
                               c64.data_ptr(), out.data_ptr(), padV, s)
    if st != 0:
        from .losses import status_string

        raise RuntimeError(f"rf_lmhead_dlogits: {status_string(st)}")
    return out[:, :V]


def lmhead_loss_and_grad(config, hidden: torch.Tensor, w_vocab: torch.Tensor, batch, stream=None,
                         check: bool = True):
    """The off-policy loss and dlogits from hidden states, logits never materialised:
    tensor-core stats sweep (lse, sampled logit) -> per-token loss math
    (``rf_token_loss_from_stats``, reference semantics) -> tensor-core dlogits sweep.

    ``batch`` is a ``losses.PackedBatch`` whose ``logits`` is only a placeholder
    (``vocab`` must be set); token_mean aggregation, no exact KL.  Returns a
    ``losses.LossResult`` (dlogits bf16 [T, V]).  ``check=False`` skips the final
    synchronisation and status check (stream-ordered use)."""
    import ctypes

    from . import losses as L

    config.validate()
    dev = hidden.device
    T = batch.num_tokens
    lse, xt = lmhead_lse(hidden, w_vocab, batch.token_ids, stream)
    f64 = torch.float64
    out = {k: torch.empty(T, dtype=f64, device=dev) for k in ("lp", "ratio", "coef", "loss")}
    flags = torch.empty(T, dtype=torch.uint8, device=dev)
    scalars = torch.zeros(_abi.RF_NUM_SCALARS, dtype=f64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    cfg_c = config.to_c()
    b = batch.to_c(0, T)
    lib = _abi.load_library()
    wsb = lib.rf_workspace_bytes(ctypes.byref(cfg_c), ctypes.byref(b))
    ws = torch.empty(max(int(wsb), 256), dtype=torch.uint8, device=dev)
    o = _abi.rf_outputs()
    o.token_logp, o.token_ratio = out["lp"].data_ptr(), out["ratio"].data_ptr()
    o.token_coef, o.token_loss, o.token_flags = out["coef"].data_ptr(), out["loss"].data_ptr(), flags.data_ptr()
    o.scalars, o.device_status = scalars.data_ptr(), status.data_ptr()
    o.workspace, o.workspace_bytes = ws.data_ptr(), ws.numel()
    s = torch.cuda.current_stream().cuda_stream if stream is None else (
        stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    st = lib.rf_token_loss_from_stats(ctypes.byref(cfg_c), ctypes.byref(b), lse.data_ptr(), xt.data_ptr(),
                                      ctypes.byref(o), s)
    if st != 0:
        raise L.InvalidArgument(L.status_string(st))
    dl = lmhead_dlogits(hidden, w_vocab, batch.token_ids, lse, out["coef"], stream)
    if check:  # synchronises, then raises like the reference (losses.cpp:267)
        torch.cuda.synchronize(dev)
        dst = int(status.item())
        if dst & _abi.RF_DEVSTAT_NONFINITE_RATIO:
            raise L.InvalidArgument(L.status_string(_abi.RF_ERR_NONFINITE_RATIO))
    return L.LossResult(scalars=scalars, dlogits=dl, token_logp=out["lp"], token_ratio=out["ratio"],
                        token_coef=out["coef"], token_loss=out["loss"], token_flags=flags)
