"""The step before the loss, fused: the LM-head GEMM on the
tensor cores with the softmax statistics in its epilogue, the reference's per-token
loss math on lp = x_tok − lse, and the backward GEMMs fed from vocabulary chunks of
dlogits — so neither the [T, V] logits nor the [T, V] dlogits tensor exists in HBM.

* ``lmhead_lse(hidden, w_vocab, token_ids)`` — ``rf_lmhead_lse`` (csrc/rf_lmhead.cu:
  TMA + 2-CTA tcgen05.mma into tensor memory, fp32 accumulation, online max/Σexp in
  the epilogue, fp64 combine across vocabulary splits): lse [T] fp64 and the sampled
  logit x_tok [T] fp32;
* ``lmhead_dlogits`` — the second tensor-core sweep writing k·(onehot − p) bf16 rows;
* ``lmhead_backward`` — dH = dlogits·W, dW = dlogitsᵀ·H chunk by chunk over the vocabulary;
* ``lmhead_loss_and_grad`` — the whole loss step from hidden states.

The logits consumer this replaces is the reference's ToyPolicy::log_probs over a
logits row (policy.cpp:21-30, called from losses.cpp:159).  Every temporary is
allocated on the launching stream (caching-allocator ordering)."""
from __future__ import annotations

import contextlib

import torch

from . import _abi


def _launch_ctx(stream):
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _handle(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(st: int, what: str) -> None:
    if st != 0:
        from .losses import status_string

        raise RuntimeError(f"{what}: {status_string(st)}")


def lmhead_lse(hidden: torch.Tensor, w_vocab: torch.Tensor, token_ids: torch.Tensor, stream=None):
    """(lse [T] fp64, x_tok [T] fp32) of logits = H·Wᵀ without materialising them."""
    if hidden.dtype != torch.bfloat16 or w_vocab.dtype != torch.bfloat16:
        raise TypeError("hidden and w_vocab must be bf16")
    if hidden.dim() != 2 or w_vocab.dim() != 2 or hidden.shape[1] != w_vocab.shape[1]:
        raise ValueError("hidden [T, K] and w_vocab [V, K] expected")
    if not (hidden.is_contiguous() and w_vocab.is_contiguous()):
        raise ValueError("row-major contiguous operands expected")
    T, K = hidden.shape
    V = w_vocab.shape[0]
    with _launch_ctx(stream):
        tok = token_ids.to(device=hidden.device, dtype=torch.int32).contiguous()
        lse = torch.empty(T, dtype=torch.float64, device=hidden.device)
        xt = torch.empty(T, dtype=torch.float32, device=hidden.device)
    _check(_abi.load_library().rf_lmhead_lse(hidden.data_ptr(), w_vocab.data_ptr(), tok.data_ptr(), T, V, K,
                                             lse.data_ptr(), xt.data_ptr(), _handle(stream)), "rf_lmhead_lse")
    return lse, xt


def lmhead_dlogits(hidden: torch.Tensor, w_vocab: torch.Tensor, token_ids: torch.Tensor, lse: torch.Tensor,
                   coef: torch.Tensor, stream=None) -> torch.Tensor:
    """dlogits[t, v] = coef[t]·(1[v = tok_t] − exp((H Wᵀ)[t, v] − lse[t])), bf16 [T, V], from a
    second tensor-core sweep (the logits are recomputed, never stored).  Token ids outside
    [0, V) contribute no one-hot term (a vocabulary chunk passes tok − v0)."""
    T, K = hidden.shape
    V = w_vocab.shape[0]
    padV = (V + 7) // 8 * 8
    with _launch_ctx(stream):
        out = torch.empty(T, padV, dtype=torch.bfloat16, device=hidden.device)
        tok = token_ids.to(device=hidden.device, dtype=torch.int32).contiguous()
        lse64 = lse.to(torch.float64).contiguous()
        c64 = coef.to(torch.float64).contiguous()
    _check(_abi.load_library().rf_lmhead_dlogits(hidden.data_ptr(), w_vocab.data_ptr(), tok.data_ptr(), T, V, K,
                                                 lse64.data_ptr(), c64.data_ptr(), out.data_ptr(), padV,
                                                 _handle(stream)), "rf_lmhead_dlogits")
    return out[:, :V]


def lmhead_backward(hidden: torch.Tensor, w_vocab: torch.Tensor, token_ids: torch.Tensor, lse: torch.Tensor,
                    coef: torch.Tensor, *, chunk_vocab: int = 24576, stream=None):
    """The LM-head backward from the loss coefficients, vocabulary chunk by chunk:

        dlogits[:, c] = coef·(1[v = tok] − exp(H·W[c]ᵀ − lse))   (tensor-core sweep, bf16)
        dH   += dlogits[:, c] · W[c]                              (cuBLAS, fp32 accumulate and output)
        dW[c] = dlogits[:, c]ᵀ · H                               (cuBLAS, fp32)

    Only one [T, chunk] dlogits tile is alive at a time, so the memory of the loss step
    does not grow with V.  The tiles are the reference's LogProbGrad rows (losses.cpp:
    87-115) restricted to the chunk; ``lse`` is the full-vocabulary lse of
    ``lmhead_lse``.  Returns (dH [T, K] fp32, dW [V, K] fp32) for the objective whose
    per-token coefficient is ``coef``.  The backward GEMMs are plain library GEMMs."""
    T, K = hidden.shape
    V = w_vocab.shape[0]
    if chunk_vocab % 256:
        raise ValueError("chunk_vocab must be a multiple of 256 (the sweep's vocabulary tile)")
    with _launch_ctx(stream):
        tok = token_ids.to(device=hidden.device, dtype=torch.int32).contiguous()
        dH = torch.zeros(T, K, dtype=torch.float32, device=hidden.device)
        dW = torch.empty(V, K, dtype=torch.float32, device=hidden.device)
        for v0 in range(0, V, chunk_vocab):
            v1 = min(V, v0 + chunk_vocab)
            wc = w_vocab[v0:v1]
            dl = lmhead_dlogits(hidden, wc, tok - v0, lse, coef, stream)
            dH += torch.mm(dl, wc, out_dtype=torch.float32)
            dW[v0:v1] = torch.mm(dl.t(), hidden, out_dtype=torch.float32)
    return dH, dW


def lmhead_loss_and_grad(config, hidden: torch.Tensor, w_vocab: torch.Tensor, batch, stream=None,
                         check: bool = True, want: str = "dlogits", chunk_vocab: int = 24576):
    """The off-policy loss from hidden states, logits never materialised: tensor-core stats
    sweep (lse, sampled logit) -> per-token loss math (``rf_token_loss_from_stats``,
    reference semantics, losses.cpp:262-331) -> either the dlogits sweep (``want="dlogits"``:
    bf16 [T, V] in ``result.dlogits``) or the chunked backward (``want="grads"``: returns
    ``(result, dH, dW)``, no [T, V] tensor at all).

    ``batch`` is a ``losses.PackedBatch`` whose ``logits`` is only a placeholder (``vocab``
    must be set); token_mean aggregation, no exact KL.  ``check=False`` skips the final
    synchronisation and status check (stream-ordered use)."""
    import ctypes

    from . import losses as L

    if want not in ("dlogits", "grads"):
        raise ValueError("want must be 'dlogits' or 'grads'")
    config.validate()
    dev = hidden.device
    T = batch.num_tokens
    lse, xt = lmhead_lse(hidden, w_vocab, batch.token_ids, stream)
    cfg_c = config.to_c()
    b = batch.to_c(0, T)
    lib = _abi.load_library()
    f64 = torch.float64
    with _launch_ctx(stream):
        out = {k: torch.empty(T, dtype=f64, device=dev) for k in ("lp", "ratio", "coef", "loss")}
        flags = torch.empty(T, dtype=torch.uint8, device=dev)
        scalars = torch.zeros(_abi.RF_NUM_SCALARS, dtype=f64, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        ws = torch.empty(max(int(lib.rf_workspace_bytes(ctypes.byref(cfg_c), ctypes.byref(b))), 256),
                         dtype=torch.uint8, device=dev)
    o = _abi.rf_outputs()
    o.token_logp, o.token_ratio = out["lp"].data_ptr(), out["ratio"].data_ptr()
    o.token_coef, o.token_loss, o.token_flags = out["coef"].data_ptr(), out["loss"].data_ptr(), flags.data_ptr()
    o.scalars, o.device_status = scalars.data_ptr(), status.data_ptr()
    o.workspace, o.workspace_bytes = ws.data_ptr(), ws.numel()
    st = lib.rf_token_loss_from_stats(ctypes.byref(cfg_c), ctypes.byref(b), lse.data_ptr(), xt.data_ptr(),
                                      ctypes.byref(o), _handle(stream))
    if st != 0:
        raise L.InvalidArgument(L.status_string(st))
    dl = dH = dW = None
    if want == "dlogits":
        dl = lmhead_dlogits(hidden, w_vocab, batch.token_ids, lse, out["coef"], stream)
    else:
        dH, dW = lmhead_backward(hidden, w_vocab, batch.token_ids, lse, out["coef"], chunk_vocab=chunk_vocab,
                                 stream=stream)
    if check:  # synchronises, then raises like the reference (losses.cpp:267)
        torch.cuda.synchronize(dev)
        dst = int(status.item())
        if dst & _abi.RF_DEVSTAT_NONFINITE_RATIO:
            raise L.InvalidArgument(L.status_string(_abi.RF_ERR_NONFINITE_RATIO))
        if dst & _abi.RF_DEVSTAT_TOKEN_OUT_OF_RANGE:
            raise L.InvalidArgument(L.status_string(_abi.RF_ERR_TOKEN_OUT_OF_RANGE))
    res = L.LossResult(scalars=scalars, dlogits=dl, token_logp=out["lp"], token_ratio=out["ratio"],
                       token_coef=out["coef"], token_loss=out["loss"], token_flags=flags, device_status=status)
    return res if want == "dlogits" else (res, dH, dW)
