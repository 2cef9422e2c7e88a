"""Batch assembly: the trainer's side of the reference's SampleBuffer, feeding the loss
directly ("SampleBuffer batch assembly feeding rf_batch").

The reference hands the trainer ``SampleBuffer::get_batch(B, consumer_version)`` —
FIFO samples whose staleness (consumer_version − init_version) it records
(sample_buffer.cpp:26-41; Sample = sample_buffer.hpp:15-23).  ``pack_samples`` turns
such a batch, plus the per-token log-probs the trainer attaches, into the packed
``PackedBatch`` of the C ABI:

* GRPO groups = the responses of one prompt (scheduler.cpp:36-41), kept whole and in
  FIFO order of their first response; sequences in FIFO order inside a group;
* with ``world > 1`` this rank's share of whole groups by LPT on group token counts
  (``dist.lpt_shard``) and the global normalisers T_global / N_global;
* one pinned host staging buffer and ONE host→device copy for all token and sequence
  arrays; the CSR offsets and ``seq_of_token`` are expanded on the device;
* the staleness histogram of the batch, as get_batch records it.

Nothing here computes the loss; the result goes to ``grpo_advantages`` and
``loss_and_grad`` / ``OffPolicyLoss``.
"""
from __future__ import annotations

from collections import Counter, OrderedDict
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from .dist import lpt_shard
from .losses import InvalidArgument, Normalization, PackedBatch


@dataclass
class Sample:
    """= rlsim::Sample (sample_buffer.hpp:15-23) plus the per-token log-probs the trainer
    attaches (behaviour policy, and optionally the proximal policy and the inference engine)."""

    prompt: int
    tokens: Sequence[int]
    reward: float
    behavior_logp: Sequence[float]
    init_version: int = 0
    id: int = 0
    prox_logp: Optional[Sequence[float]] = None
    engine_logp: Optional[Sequence[float]] = None


@dataclass
class PackInfo:
    global_num_tokens: int
    global_num_seqs: int
    num_groups: int
    sample_ids: List[int]                       # this rank's samples, in packed order
    staleness_histogram: Dict[int, int] = field(default_factory=dict)


def pack_samples(samples: Sequence[Sample], logits: Optional[torch.Tensor] = None, *, consumer_version: int = 0,
                 rank: int = 0, world: int = 1, device="cuda", normalization=Normalization.global_token,
                 grad_sign: float = 1.0, vocab: Optional[int] = None, row_of_token: Optional[torch.Tensor] = None):
    """Pack a get_batch() result into (PackedBatch, PackInfo) for this rank.

    ``logits`` are this rank's rows in packed token order ([T_rank, >= V], one row per
    token: the LM head's output), or a pool indexed by ``row_of_token``; ``None`` leaves a
    placeholder (set ``vocab``) for the LM-head path.  Log-prob arrays go to the device as
    f32.  Raises InvalidArgument for an empty batch, an empty trajectory, mismatched
    log-prob lengths or a group of < 2 responses (losses.cpp:42,140,157)."""
    if len(samples) == 0:
        raise InvalidArgument("loss_and_grad: empty batch")
    groups: "OrderedDict[int, List[Sample]]" = OrderedDict()
    for s in samples:
        if len(s.tokens) == 0:
            raise InvalidArgument("loss_and_grad: empty trajectory")
        if len(s.behavior_logp) != len(s.tokens):
            raise InvalidArgument("trajectory_ratio: behavior log-probs missing")
        for name in ("prox_logp", "engine_logp"):
            v = getattr(s, name)
            if v is not None and len(v) != len(s.tokens):
                raise InvalidArgument(f"pack_samples: {name} length differs from the tokens")
        groups.setdefault(int(s.prompt), []).append(s)
    if any(len(g) < 2 for g in groups.values()):
        raise InvalidArgument("grpo_advantages: group size must be >= 2")
    glist = list(groups.values())
    gtok = [sum(len(s.tokens) for s in g) for g in glist]
    mine = lpt_shard(gtok, world)[rank] if world > 1 else list(range(len(glist)))
    if not mine:
        raise InvalidArgument(f"pack_samples: rank {rank} of {world} owns no group")
    seqs = [s for gi in mine for s in glist[gi]]
    has_prox = all(s.prox_logp is not None for s in seqs)
    has_eng = all(s.engine_logp is not None for s in seqs)
    lens = np.array([len(s.tokens) for s in seqs], dtype=np.int64)
    T, N = int(lens.sum()), len(seqs)
    # one staging buffer: [lengths i64 | rewards f64 | group sizes i64 | tokens i32 | behavior f32 | prox f32 |
    # engine f32] (8-byte arrays first, so every view is aligned)
    nlp = 1 + int(has_prox) + int(has_eng)
    G = len(mine)
    nbytes = T * 4 * (1 + nlp) + N * 8 * 2 + G * 8
    on_cuda = torch.device(device).type == "cuda"
    stage = torch.empty(nbytes, dtype=torch.uint8, pin_memory=on_cuda)
    buf = stage.numpy()
    off = 0

    def view(n, dt):
        nonlocal off
        v = buf[off:off + n * np.dtype(dt).itemsize].view(dt)
        off += n * np.dtype(dt).itemsize
        return v

    lv, rew, gs = view(N, np.int64), view(N, np.float64), view(G, np.int64)
    tok, beh = view(T, np.int32), view(T, np.float32)
    prox = view(T, np.float32) if has_prox else None
    eng = view(T, np.float32) if has_eng else None
    pos = 0
    for i, s in enumerate(seqs):
        n = len(s.tokens)
        tok[pos:pos + n] = s.tokens
        beh[pos:pos + n] = s.behavior_logp
        if prox is not None:
            prox[pos:pos + n] = s.prox_logp
        if eng is not None:
            eng[pos:pos + n] = s.engine_logp
        rew[i] = s.reward
        pos += n
    lv[:] = lens
    gs[:] = [len(glist[gi]) for gi in mine]
    d = stage.to(device, non_blocking=on_cuda)  # the one host -> device copy

    def dview(start, n, dt):
        return d[start:start + n * torch.tensor([], dtype=dt).element_size()].view(dt)

    o = 0
    d_len = dview(o, N, torch.int64)
    o += N * 8
    d_rew = dview(o, N, torch.float64)
    o += N * 8
    d_gs = dview(o, G, torch.int64)
    o += G * 8
    d_tok = dview(o, T, torch.int32)
    o += T * 4
    d_beh = dview(o, T, torch.float32)
    o += T * 4
    d_prox = d_eng = None
    if has_prox:
        d_prox = dview(o, T, torch.float32)
        o += T * 4
    if has_eng:
        d_eng = dview(o, T, torch.float32)
    seq_offsets = torch.zeros(N + 1, dtype=torch.int64, device=device)
    torch.cumsum(d_len, 0, out=seq_offsets[1:])
    group_offsets = torch.zeros(G + 1, dtype=torch.int64, device=device)
    torch.cumsum(d_gs, 0, out=group_offsets[1:])
    if logits is None:
        if vocab is None:
            raise InvalidArgument("pack_samples: vocab is required without logits")
        logits = torch.empty(1, vocab, dtype=torch.bfloat16, device=device)  # placeholder (LM-head path)
    pb = PackedBatch(logits=logits, token_ids=d_tok, seq_offsets=seq_offsets, advantages=None, behavior_logp=d_beh,
                     vocab=vocab, row_of_token=row_of_token, prox_logp=d_prox, engine_logp=d_eng, rewards=d_rew,
                     group_offsets=group_offsets, normalization=normalization,
                     global_num_seqs=len(samples), global_num_tokens=int(sum(gtok)), grad_sign=grad_sign)
    hist = Counter(int(consumer_version - s.init_version) for s in seqs)
    info = PackInfo(global_num_tokens=int(sum(gtok)), global_num_seqs=len(samples), num_groups=G,
                    sample_ids=[int(s.id) for s in seqs], staleness_histogram=dict(sorted(hist.items())))
    return pb, info
