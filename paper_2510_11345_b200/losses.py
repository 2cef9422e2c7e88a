"""Host-side mirror of the reference loss interface over the CUDA C ABI.

Two layers, both thin Python over ``librf_offpolicy.so``:

* the packed LLM-layout API (``PackedBatch`` + ``loss_and_grad`` /
  ``grpo_advantages`` / ``OffPolicyLoss``): device tensors in, per-token dlogits
  and diagnostics out, stream-ordered;
* the rlsim-shaped API (``LossVariant``, ``LossConfig``, ``Trajectory``,
  ``loss_and_grad_policy``): the same names, argument meaning and error
  behaviour as ``rlsim::loss_and_grad`` (reference proj/include/rlsim/losses.hpp:
  10-78), so a caller of the reference can switch by changing the import.

Errors mirror the reference's ``std::invalid_argument`` throw sites
(losses.cpp:29,33-38,140-174,205,267) as ``InvalidArgument`` with the same
messages.  Nothing here computes the loss on the CPU.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _abi
from ._abi import rf_batch, rf_loss_config, rf_outputs


class InvalidArgument(ValueError):
    """Mirror of the reference's std::invalid_argument."""


class LossVariant(enum.IntEnum):
    """= rlsim::LossVariant (losses.hpp:10-18)."""

    ppo = 0
    decoupled_ppo = 1
    tis = 2
    cispo = 3
    topr = 4
    grpo = 5
    naive_is = 6


class RatioAggregation(enum.IntEnum):
    """= rlsim::RatioAggregation (losses.hpp:23-26)."""

    token_mean = 0
    sequence_product = 1


class Normalization(enum.IntEnum):
    seq_then_batch = _abi.RF_NORM_SEQ_THEN_BATCH
    global_token = _abi.RF_NORM_GLOBAL_TOKEN


def _lib():
    return _abi.load_library()


def to_string(v: int) -> str:
    """rlsim::to_string(LossVariant) (losses.cpp:8-19)."""
    return _lib().rf_loss_variant_name(int(v)).decode()


def loss_variant_from_string(s: str) -> LossVariant:
    """rlsim::loss_variant_from_string (losses.cpp:21-30)."""
    out = ctypes.c_int32(0)
    st = _lib().rf_loss_variant_from_name(s.encode(), ctypes.byref(out))
    if st != _abi.RF_OK:
        raise InvalidArgument("unknown loss variant: " + s)
    return LossVariant(out.value)


def status_string(st: int) -> str:
    return _lib().rf_status_string(int(st)).decode()


def _raise_for(st: int) -> None:
    if st != _abi.RF_OK:
        raise InvalidArgument(status_string(st)) if st != _abi.RF_ERR_CUDA else RuntimeError(status_string(st))


@dataclass
class LossConfig:
    """= rlsim::LossConfig (losses.hpp:28-41), same defaults."""

    variant: LossVariant = LossVariant.ppo
    clip_eps: float = 0.2
    eps_low: float = 0.2
    eps_high: float = 0.2
    trunc_cap: float = 5.0
    kl_weight: float = 0.0
    w_plus: float = 1.0
    w_minus: float = 1.0
    engine_mismatch_cap: float = 0.0
    aggregation: RatioAggregation = RatioAggregation.token_mean

    def to_c(self) -> rf_loss_config:
        return rf_loss_config(
            int(self.variant), int(self.aggregation), float(self.clip_eps), float(self.eps_low),
            float(self.eps_high), float(self.trunc_cap), float(self.kl_weight), float(self.w_plus),
            float(self.w_minus), float(self.engine_mismatch_cap),
        )

    def validate(self) -> None:
        """LossConfig::validate (losses.cpp:32-39): raises InvalidArgument."""
        c = self.to_c()
        _raise_for(_lib().rf_loss_config_validate(ctypes.byref(c)))


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


_DT = {torch.bfloat16: _abi.RF_DTYPE_BF16, torch.float32: _abi.RF_DTYPE_F32, torch.float64: _abi.RF_DTYPE_F64}


def seq_of_token_from_offsets(seq_offsets: torch.Tensor) -> torch.Tensor:
    """Per-token sequence index from CSR offsets (int32)."""
    offs = seq_offsets.to(torch.int64)
    lens = offs[1:] - offs[:-1]
    return torch.repeat_interleave(torch.arange(lens.numel(), device=offs.device, dtype=torch.int32), lens)


@dataclass
class PackedBatch:
    """A packed ragged batch on the GPU (see include/rf_offpolicy.h rf_batch).

    One reference ``Trajectory`` (policy.hpp:44-51) = one CSR sequence; its
    ``context`` row = ``row_of_token`` of its tokens (None -> one row per token).
    """

    logits: torch.Tensor                 # [rows, >= vocab] bf16 | f32
    token_ids: torch.Tensor              # [T] int32
    seq_offsets: torch.Tensor            # [N+1] int64
    advantages: Optional[torch.Tensor]   # [N] f64
    behavior_logp: torch.Tensor          # [T] f32 | f64
    vocab: Optional[int] = None
    seq_of_token: Optional[torch.Tensor] = None   # [T] int32
    row_of_token: Optional[torch.Tensor] = None   # [T] int32
    prox_logp: Optional[torch.Tensor] = None
    engine_logp: Optional[torch.Tensor] = None
    ref_logits: Optional[torch.Tensor] = None
    rewards: Optional[torch.Tensor] = None        # [N] f64
    group_offsets: Optional[torch.Tensor] = None  # [G+1] int64
    normalization: Normalization = Normalization.seq_then_batch
    global_num_seqs: Optional[int] = None
    global_num_tokens: Optional[int] = None
    grad_sign: float = 1.0

    def __post_init__(self):
        if self.vocab is None:
            self.vocab = int(self.logits.shape[-1])
        if self.seq_of_token is None:
            self.seq_of_token = seq_of_token_from_offsets(self.seq_offsets)
        if self.global_num_seqs is None:
            self.global_num_seqs = int(self.seq_offsets.numel() - 1)
        if self.global_num_tokens is None:
            self.global_num_tokens = int(self.token_ids.numel())

    @property
    def num_tokens(self) -> int:
        return int(self.token_ids.numel())

    @property
    def num_seqs(self) -> int:
        return int(self.seq_offsets.numel() - 1)

    def sequence_chunks(self, max_tokens: int):
        """Split into calls of whole sequences (sequence_product needs every token of
        a sequence in one call).  Yields (t0, t1, sub_batch): the sub-batch views the
        token arrays [t0, t1), the sequence arrays of its sequences, and has
        ``seq_of_token`` rebased to them; global normalisers are kept."""
        offs = self.seq_offsets.cpu().tolist()
        N = len(offs) - 1
        s = 0
        while s < N:
            e = s + 1
            while e < N and offs[e + 1] - offs[s] <= max_tokens:
                e += 1
            t0, t1 = offs[s] - offs[0], offs[e] - offs[0]
            sub = PackedBatch(
                logits=self.logits if self.row_of_token is not None else self.logits[t0:t1],
                token_ids=self.token_ids[t0:t1], seq_offsets=self.seq_offsets[s:e + 1],
                advantages=None if self.advantages is None else self.advantages[s:e],
                behavior_logp=self.behavior_logp[t0:t1], vocab=self.vocab,
                seq_of_token=self.seq_of_token[t0:t1] - s,
                row_of_token=None if self.row_of_token is None else self.row_of_token[t0:t1],
                prox_logp=None if self.prox_logp is None else self.prox_logp[t0:t1],
                engine_logp=None if self.engine_logp is None else self.engine_logp[t0:t1],
                ref_logits=(self.ref_logits if (self.ref_logits is None or self.row_of_token is not None)
                            else self.ref_logits[t0:t1]),
                normalization=self.normalization, global_num_seqs=self.global_num_seqs,
                global_num_tokens=self.global_num_tokens, grad_sign=self.grad_sign)
            yield t0, t1, sub
            s = e

    def to_c(self, t0: int = 0, t1: Optional[int] = None) -> rf_batch:
        """rf_batch for the token range [t0, t1) (a streaming chunk)."""
        T = self.num_tokens
        t1 = T if t1 is None else t1
        lp_dt = _DT[self.behavior_logp.dtype]
        es_lp = self.behavior_logp.element_size()
        b = rf_batch()
        b.num_tokens = t1 - t0
        b.num_seqs = self.num_seqs
        b.num_groups = 0 if self.group_offsets is None else int(self.group_offsets.numel() - 1)
        b.vocab = int(self.vocab)
        b.logits_dtype = _DT[self.logits.dtype]
        b.logits = self.logits.data_ptr()
        b.logits_row_stride = int(self.logits.stride(0))
        b.row_of_token = None if self.row_of_token is None else self.row_of_token.data_ptr() + 4 * t0
        if self.row_of_token is None and t0:
            b.logits = self.logits.data_ptr() + t0 * self.logits.stride(0) * self.logits.element_size()
        b.token_ids = self.token_ids.data_ptr() + 4 * t0
        b.seq_of_token = self.seq_of_token.data_ptr() + 4 * t0
        b.seq_offsets = self.seq_offsets.data_ptr()
        b.group_offsets = _ptr(self.group_offsets)
        b.rewards = _ptr(self.rewards)
        b.advantages = _ptr(self.advantages)
        b.logp_dtype = lp_dt
        b.normalization = int(self.normalization)
        b.behavior_logp = self.behavior_logp.data_ptr() + es_lp * t0
        b.prox_logp = None if self.prox_logp is None else self.prox_logp.data_ptr() + es_lp * t0
        b.engine_logp = None if self.engine_logp is None else self.engine_logp.data_ptr() + es_lp * t0
        if self.ref_logits is not None:
            off = 0 if self.row_of_token is not None else t0 * self.ref_logits.stride(0) * self.ref_logits.element_size()
            b.ref_logits = self.ref_logits.data_ptr() + off
            b.ref_row_stride = int(self.ref_logits.stride(0))
        b.global_num_seqs = int(self.global_num_seqs)
        b.global_num_tokens = int(self.global_num_tokens)
        b.grad_sign = float(self.grad_sign)
        return b


@dataclass
class LossResult:
    """Outputs of one loss_and_grad call (device tensors)."""

    scalars: torch.Tensor
    dlogits: Optional[torch.Tensor] = None
    token_logp: Optional[torch.Tensor] = None
    token_ratio: Optional[torch.Tensor] = None
    token_coef: Optional[torch.Tensor] = None
    token_loss: Optional[torch.Tensor] = None
    token_flags: Optional[torch.Tensor] = None
    device_status: Optional[torch.Tensor] = None
    launches: int = 0

    @property
    def value(self) -> float:
        return float(self.scalars[_abi.RF_SCALAR_LOSS])


def _stream_handle(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def grpo_advantages(rewards: torch.Tensor, group_offsets: torch.Tensor, stream=None, *, out=None,
                    validate: bool = True):
    """K1 — rlsim::grpo_advantages (losses.cpp:41-60) over CSR groups on the GPU.

    Returns (advantages f64 [N], degenerate uint8 [G]).  Bit-identical to the
    reference.  Raises InvalidArgument for a group smaller than 2, as the reference
    does (losses.cpp:42): ``validate`` checks the offsets on the host before the
    launch and the device status after it.  A training loop validates its batch
    layout once and passes ``validate=False`` plus preallocated ``out=(adv, deg,
    status)`` to keep the step free of host syncs and allocations; the kernel then
    ORs RF_DEVSTAT_GROUP_TOO_SMALL into ``status`` (and zeroes that group's
    advantages) for the caller to read later.
    """
    G = int(group_offsets.numel() - 1)
    if G <= 0:
        raise InvalidArgument("grpo_advantages: group size must be >= 2")
    if validate:
        sizes = (group_offsets[1:] - group_offsets[:-1])
        if bool((sizes < 2).any()):
            raise InvalidArgument("grpo_advantages: group size must be >= 2")
    dev = rewards.device
    if stream is not None:
        ctx = torch.cuda.stream(stream)
    else:
        import contextlib
        ctx = contextlib.nullcontext()
    with ctx:  # temporaries belong to the launching stream (caching-allocator ordering)
        if out is not None:
            adv, deg, status = out
        else:
            adv = torch.empty_like(rewards, dtype=torch.float64)
            deg = torch.empty(G, dtype=torch.uint8, device=dev)
            status = torch.zeros(1, dtype=torch.int32, device=dev)
    b = rf_batch()
    b.num_groups = G
    b.num_seqs = int(rewards.numel())
    b.rewards = rewards.data_ptr()
    b.group_offsets = group_offsets.data_ptr()
    o = rf_outputs()
    o.advantages_out = adv.data_ptr()
    o.group_degenerate = deg.data_ptr()
    o.device_status = status.data_ptr()
    _raise_for(_lib().rf_grpo_advantages(ctypes.byref(b), ctypes.byref(o), _stream_handle(stream)))
    if validate and int(status.item()) & _abi.RF_DEVSTAT_GROUP_TOO_SMALL:
        raise InvalidArgument("grpo_advantages: group size must be >= 2")
    return adv, deg


_KERNEL = {"auto": _abi.RF_KERNEL_AUTO, "ring": _abi.RF_KERNEL_RING, "generic": _abi.RF_KERNEL_GENERIC}


class OffPolicyLoss:
    """Preallocated outputs + workspace for repeated (chunked) calls.

    ``run(batch, t0, t1)`` launches K2(+K3) for tokens [t0, t1) into the
    preallocated buffers without synchronising (the streaming/bench path).
    """

    def __init__(self, config: LossConfig, batch: PackedBatch, *, chunk_tokens: Optional[int] = None,
                 dlogits_dtype=torch.bfloat16, want_dlogits: bool = True, want_token_outputs: bool = True,
                 kernel: str = "auto"):
        config.validate()
        self.config = config
        self.cfg_c = config.to_c()
        self.kernel = _KERNEL[kernel]
        dev = batch.logits.device
        T = batch.num_tokens
        self.chunk = T if chunk_tokens is None else min(int(chunk_tokens), T)
        V = int(batch.vocab)
        pad = (V + 7) // 8 * 8
        self.dlogits = (torch.empty(self.chunk, pad, dtype=dlogits_dtype, device=dev)[:, :V]
                        if want_dlogits else None)
        f64 = torch.float64
        self.token_logp = torch.empty(T, dtype=f64, device=dev) if want_token_outputs else None
        self.token_ratio = torch.empty(T, dtype=f64, device=dev) if want_token_outputs else None
        self.token_coef = torch.empty(T, dtype=f64, device=dev) if want_token_outputs else None
        self.token_loss = torch.empty(T, dtype=f64, device=dev) if want_token_outputs else None
        self.token_flags = torch.empty(T, dtype=torch.uint8, device=dev) if want_token_outputs else None
        self.scalars = torch.zeros(_abi.RF_NUM_SCALARS, dtype=f64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        probe = batch.to_c(0, self.chunk)
        wsb = _lib().rf_workspace_bytes(ctypes.byref(self.cfg_c), ctypes.byref(probe))
        self.workspace = torch.empty(max(int(wsb), 256), dtype=torch.uint8, device=dev)
        self.launches = 0

    def outputs_c(self, t0: int) -> rf_outputs:
        o = rf_outputs()
        if self.dlogits is not None:
            o.dlogits = self.dlogits.data_ptr()
            o.dlogits_dtype = _DT[self.dlogits.dtype]
            o.dlogits_row_stride = int(self.dlogits.stride(0))
        if self.token_logp is not None:
            o.token_logp = self.token_logp.data_ptr() + 8 * t0
            o.token_ratio = self.token_ratio.data_ptr() + 8 * t0
            o.token_coef = self.token_coef.data_ptr() + 8 * t0
            o.token_loss = self.token_loss.data_ptr() + 8 * t0
            o.token_flags = self.token_flags.data_ptr() + t0
        o.scalars = self.scalars.data_ptr()
        o.device_status = self.status.data_ptr()
        o.workspace = self.workspace.data_ptr()
        o.workspace_bytes = self.workspace.numel()
        return o

    def zero(self, stream=None) -> None:
        o = self.outputs_c(0)
        _raise_for(_lib().rf_zero_scalars(ctypes.byref(o), _stream_handle(stream)))

    def run(self, batch: PackedBatch, t0: int = 0, t1: Optional[int] = None, stream=None,
            out_t0: Optional[int] = None) -> None:
        """Tokens [t0, t1) of ``batch``; per-token outputs land at ``out_t0`` (default t0)
        of the preallocated arrays (a sequence chunk from ``sequence_chunks`` passes its
        own offset)."""
        t1 = batch.num_tokens if t1 is None else t1
        if t1 - t0 > self.chunk:
            raise InvalidArgument("chunk larger than the preallocated dlogits buffer")
        b = batch.to_c(t0, t1)
        o = self.outputs_c(t0 if out_t0 is None else out_t0)
        lib = _lib()
        _raise_for(lib.rf_loss_and_grad_ex(ctypes.byref(self.cfg_c), ctypes.byref(b), ctypes.byref(o),
                                           _stream_handle(stream), self.kernel))
        self.launches += int(lib.rf_last_launch_count())


def loss_and_grad(config: LossConfig, batch: PackedBatch, *, dlogits_dtype=torch.bfloat16,
                  want_dlogits: bool = True, kernel: str = "auto", stream=None,
                  check: bool = True) -> LossResult:
    """rlsim::loss_and_grad (losses.cpp:137-331) on a packed GPU batch.

    One fused pass (K2 + K3) over all tokens; returns per-token dlogits and
    diagnostics.  With ``check`` the call synchronises and raises
    InvalidArgument on a non-finite ratio, as the reference does
    (losses.cpp:205,267).
    """
    if stream is not None:
        with torch.cuda.stream(stream):  # outputs + workspace belong to the launching stream
            op = OffPolicyLoss(config, batch, dlogits_dtype=dlogits_dtype, want_dlogits=want_dlogits, kernel=kernel)
    else:
        op = OffPolicyLoss(config, batch, dlogits_dtype=dlogits_dtype, want_dlogits=want_dlogits, kernel=kernel)
    op.zero(stream)
    op.run(batch, 0, batch.num_tokens, stream)
    res = LossResult(scalars=op.scalars, dlogits=op.dlogits, token_logp=op.token_logp,
                     token_ratio=op.token_ratio, token_coef=op.token_coef, token_loss=op.token_loss,
                     token_flags=op.token_flags, device_status=op.status, launches=op.launches)
    if check:
        torch.cuda.synchronize(batch.logits.device)
        st = int(op.status.item())
        if st & _abi.RF_DEVSTAT_NONFINITE_RATIO:
            raise InvalidArgument("loss_and_grad: non-finite ratio")
        if st & _abi.RF_DEVSTAT_TOKEN_OUT_OF_RANGE:
            raise InvalidArgument(status_string(_abi.RF_ERR_TOKEN_OUT_OF_RANGE))
        if st & _abi.RF_DEVSTAT_EMPTY_TRAJECTORY:
            raise InvalidArgument("loss_and_grad: empty trajectory")
    return res


# ---------------------------------------------------------------------------
# rlsim-shaped API: Trajectory + tabular policy (mapping B), reference semantics.
# ---------------------------------------------------------------------------
@dataclass
class Trajectory:
    """= rlsim::Trajectory (policy.hpp:44-51)."""

    context: int = 0
    tokens: Sequence[int] = field(default_factory=list)
    reward: float = 0.0
    advantage: float = 0.0
    behavior_logp: Sequence[float] = field(default_factory=list)
    engine_logp: Sequence[float] = field(default_factory=list)


@dataclass
class PolicyLossResult:
    """= rlsim::LossResult (losses.hpp:59-63): value and grad [C*V] (host fp64)."""

    value: float
    grad: "torch.Tensor"
    used_degenerate_group: bool = False


def loss_and_grad_policy(config: LossConfig, policy_logits, batch: Sequence[Trajectory], *, prox_logits=None,
                         ref_logits=None, device: int = 0) -> PolicyLossResult:
    """Drop-in for rlsim::loss_and_grad(config, ToyPolicy, batch, LossInputs).

    ``policy_logits`` / ``prox_logits`` / ``ref_logits`` are [contexts, vocab]
    tables (ToyPolicy::logits, row-major).  The tables go to the GPU as f32
    rows; every trajectory becomes one CSR sequence whose tokens read its
    context row ("mapping B"), normalised 1/(N*L_i) exactly as the reference.
    The proximal policy's per-token log-probs are computed by a GPU pass of the
    same kernel over the prox table.  grad is the per-context sum of the
    per-token fp32 dlogits rows, accumulated in fp64 on the GPU.
    """
    config.validate()
    if len(batch) == 0:
        raise InvalidArgument("loss_and_grad: empty batch")
    if config.variant == LossVariant.decoupled_ppo and prox_logits is None:
        raise InvalidArgument("loss_and_grad: decoupled_ppo requires a proximal policy")
    if config.variant == LossVariant.grpo and config.kl_weight > 0.0 and ref_logits is None:
        raise InvalidArgument("loss_and_grad: grpo with kl_weight > 0 requires a reference policy")
    for t in batch:
        if len(t.tokens) == 0:
            raise InvalidArgument("loss_and_grad: empty trajectory")
        if config.engine_mismatch_cap > 0.0 and len(t.engine_logp) != len(t.tokens):
            raise InvalidArgument("loss_and_grad: engine log-probs missing for mismatch correction")
    dev = torch.device("cuda", device)
    tab = torch.as_tensor(policy_logits, dtype=torch.float64)
    C, V = int(tab.shape[0]), int(tab.shape[1])
    pad = (V + 3) // 4 * 4

    def table(x):
        t = torch.zeros(C, pad, dtype=torch.float32, device=dev)
        t[:, :V] = torch.as_tensor(x, dtype=torch.float64).reshape(C, V).to(dev, torch.float32)
        return t[:, :V]

    logits = table(tab)
    lens = [len(t.tokens) for t in batch]
    offs = torch.zeros(len(batch) + 1, dtype=torch.int64)
    offs[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int64), 0)
    tokens = torch.tensor([tok for t in batch for tok in t.tokens], dtype=torch.int32)
    rows = torch.tensor([t.context for t in batch for _ in t.tokens], dtype=torch.int32)
    if bool(((tokens < 0) | (tokens >= V)).any()) or bool(((rows < 0) | (rows >= C)).any()):
        raise InvalidArgument(status_string(_abi.RF_ERR_TOKEN_OUT_OF_RANGE))
    beh = torch.tensor([b for t in batch for b in t.behavior_logp], dtype=torch.float64)
    if beh.numel() != tokens.numel():
        raise InvalidArgument("trajectory_ratio: behavior log-probs missing")
    eng = (torch.tensor([e for t in batch for e in t.engine_logp], dtype=torch.float64)
           if config.engine_mismatch_cap > 0.0 else None)
    adv = torch.tensor([t.advantage for t in batch], dtype=torch.float64)
    pb = PackedBatch(logits=logits, token_ids=tokens.to(dev), seq_offsets=offs.to(dev), advantages=adv.to(dev),
                     behavior_logp=beh.to(dev), row_of_token=rows.to(dev),
                     engine_logp=None if eng is None else eng.to(dev),
                     normalization=Normalization.seq_then_batch)
    if prox_logits is not None and config.variant == LossVariant.decoupled_ppo:
        # per-token prox log-probs: a stats-only GPU pass over the prox table
        pq = PackedBatch(logits=table(prox_logits), token_ids=pb.token_ids, seq_offsets=pb.seq_offsets,
                         advantages=pb.advantages, behavior_logp=pb.behavior_logp, row_of_token=pb.row_of_token,
                         normalization=Normalization.seq_then_batch)
        qres = loss_and_grad(LossConfig(variant=LossVariant.naive_is), pq, want_dlogits=False, check=False)
        pb.prox_logp = qres.token_logp.clone()
    if ref_logits is not None and config.variant == LossVariant.grpo and config.kl_weight > 0.0:
        pb.ref_logits = table(ref_logits)
    res = loss_and_grad(config, pb, dlogits_dtype=torch.float32)
    # LossResult.grad: per-context fp64 sums of the per-token dlogits rows in token order
    # (rf_rows_segment_sum, deterministic — LogProbGrad's per-context accumulation, losses.cpp:87-115)
    order = torch.argsort(rows, stable=True)
    seg = torch.zeros(C + 1, dtype=torch.int64)
    seg[1:] = torch.cumsum(torch.bincount(rows.to(torch.int64), minlength=C), 0)
    d_seg, d_idx = seg.to(dev), order.to(torch.int32).to(dev)
    grad = torch.empty(C, V, dtype=torch.float64, device=dev)
    _raise_for(_lib().rf_rows_segment_sum(res.dlogits.data_ptr(), _abi.RF_DTYPE_F32, int(res.dlogits.stride(0)),
                                          d_seg.data_ptr(), d_idx.data_ptr(), C, V, grad.data_ptr(), V,
                                          _stream_handle(None)))
    return PolicyLossResult(value=res.value, grad=grad.reshape(-1).cpu())
