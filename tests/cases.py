"""Seeded case builders shared by the parity tests (CPU side, numpy)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_2510_11345_b200.losses import LossConfig, LossVariant, RatioAggregation


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 values to the nearest bf16 (RNE), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def log_softmax_rows(x: np.ndarray) -> np.ndarray:
    m = x.max(axis=1, keepdims=True)
    return x - (m + np.log(np.exp(x - m).sum(axis=1, keepdims=True)))


@dataclass
class Case:
    """A packed batch on the host (float64 logits already bf16/f32-representable)."""

    logits: np.ndarray            # [R, V]
    token_ids: np.ndarray         # [T] int32
    seq_offsets: np.ndarray       # [N+1] int64
    advantages: np.ndarray        # [N]
    behavior_logp: np.ndarray     # [T]
    row_of_token: Optional[np.ndarray] = None
    prox_logp: Optional[np.ndarray] = None
    engine_logp: Optional[np.ndarray] = None
    ref_logits: Optional[np.ndarray] = None
    rewards: Optional[np.ndarray] = None
    group_offsets: Optional[np.ndarray] = None

    @property
    def T(self):
        return len(self.token_ids)

    @property
    def N(self):
        return len(self.seq_offsets) - 1

    @property
    def V(self):
        return self.logits.shape[1]


def make_case(seed: int, *, T_seqs: int, G: int, V: int, max_len: int, mapping: str = "A", scale: float = 2.0,
              stale: float = 0.05, alpha: int = 2, round_bf16: bool = True, prox_table: bool = False,
              kl: bool = False, engine: bool = True) -> Case:
    """Random GRPO batch: T_seqs//G groups of G sequences with ragged lengths.

    mapping "A": every token owns its logits row (LLM layout);
    mapping "B": every sequence's tokens share one row (reference ToyPolicy layout).
    """
    rng = np.random.default_rng(seed)
    N = T_seqs
    lens = np.minimum(np.ceil(np.exp(rng.normal(np.log(max(max_len / 8, 1)), 1.0, N))), max_len).astype(np.int64)
    lens = np.maximum(lens, 1)
    offs = np.zeros(N + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    T = int(offs[-1])
    R = T if mapping == "A" else N
    logits = rng.normal(0.0, scale, (R, V))
    if round_bf16:
        logits = bf16_round(logits)
    rows = None if mapping == "A" else np.repeat(np.arange(N, dtype=np.int32), lens)
    lp_all = log_softmax_rows(logits)
    row_idx = np.arange(T) if rows is None else rows
    # tokens drawn from the row's softmax (Gumbel-max)
    g = rng.gumbel(size=(R, V)) if mapping == "A" else None
    if mapping == "A":
        tok = np.argmax(logits + g, axis=1).astype(np.int32)
    else:
        tok = np.empty(T, dtype=np.int32)
        for i in range(N):
            p = np.exp(lp_all[i])
            tok[offs[i]:offs[i + 1]] = rng.choice(V, size=lens[i], p=p / p.sum())
    lp = lp_all[row_idx, tok]
    s = rng.integers(0, alpha + 1, N)
    delta = rng.normal(0.0, 1.0, T) * stale * np.sqrt(np.repeat(s, lens))
    behavior = lp - delta
    prox = lp - delta / 2
    eng = behavior - rng.normal(0.0, 0.01, T) if engine else None
    G = max(G, 2)
    ngroups = N // G
    go = np.arange(ngroups + 1, dtype=np.int64) * G
    go[-1] = N
    p_prompt = rng.uniform(0, 1, ngroups)
    rewards = (rng.uniform(0, 1, N) < np.repeat(p_prompt, np.diff(go))).astype(np.float64)
    adv = np.zeros(N)
    for gi in range(ngroups):
        r = rewards[go[gi]:go[gi + 1]]
        mean = r.sum() / len(r)
        sd = np.sqrt(((r - mean) ** 2).sum() / len(r))
        if sd >= 1e-8:
            adv[go[gi]:go[gi + 1]] = (r - mean) / sd
    ref = None
    if kl:
        ref = logits + rng.normal(0.0, 0.3, logits.shape)
        if round_bf16:
            ref = bf16_round(ref)
    return Case(logits=logits, token_ids=tok, seq_offsets=offs, advantages=adv, behavior_logp=behavior,
                row_of_token=rows, prox_logp=prox, engine_logp=eng, ref_logits=ref, rewards=rewards,
                group_offsets=go)


def make_pool_case(seed: int, *, V: int, R: int, T_min: int, G: int = 8, max_len: int = 64, scale: float = 2.0,
                   stale: float = 0.2, alpha: int = 2, round_bf16: bool = True, kl: bool = False,
                   mapping: str = "A", draws: int = 16) -> Case:
    """A batch shaped like the benchmark's DeviceWorkload (synth.py): a pool of R
    logits rows and at least T_min tokens whose rows wrap the pool
    (row_of_token[t] = t mod R), each token drawn from its row's softmax (draw
    (t div R) mod ``draws`` of the row).  mapping "B": every sequence reads one pool
    row (its context).  Sizes are chosen so a persistent kernel gets many rows per
    CTA / cluster while the fp64 oracle stays at seconds."""
    rng = np.random.default_rng(seed)
    lens = []
    while sum(lens) < T_min or len(lens) % G:
        lens.append(int(min(max_len, max(1, np.ceil(np.exp(rng.normal(np.log(max(max_len / 8, 1)), 1.0)))))))
    lens = np.array(lens, dtype=np.int64)
    N = len(lens)
    offs = np.zeros(N + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    T = int(offs[-1])
    logits = rng.normal(0.0, scale, (R, V))
    if round_bf16:
        logits = bf16_round(logits)
    lp_all = log_softmax_rows(logits)
    p_all = np.exp(lp_all)
    tab = np.stack([rng.choice(V, size=draws, p=p_all[r] / p_all[r].sum()) for r in range(R)]).astype(np.int32)
    del p_all
    t = np.arange(T)
    if mapping == "A":
        rows = (t % R).astype(np.int32)
        tok = tab[rows, (t // R) % draws]
    else:
        seq = np.repeat(np.arange(N), lens)
        rows = (seq % R).astype(np.int32)
        tok = tab[rows, (t - offs[seq]) % draws]
    lp = lp_all[rows, tok]
    s = rng.integers(0, alpha + 1, N)
    delta = rng.normal(0.0, 1.0, T) * stale * np.sqrt(np.repeat(s, lens))
    behavior = lp - delta
    prox = lp - delta / 2
    eng = behavior - rng.normal(0.0, 0.01, T)
    ngroups = N // G
    go = np.arange(ngroups + 1, dtype=np.int64) * G
    p_prompt = rng.uniform(0, 1, ngroups)
    rewards = (rng.uniform(0, 1, N) < np.repeat(p_prompt, G)).astype(np.float64)
    adv = np.zeros(N)
    for gi in range(ngroups):
        r = rewards[go[gi]:go[gi + 1]]
        mean = r.sum() / len(r)
        sd = np.sqrt(((r - mean) ** 2).sum() / len(r))
        if sd >= 1e-8:
            adv[go[gi]:go[gi + 1]] = (r - mean) / sd
    ref = None
    if kl:
        ref = logits + rng.normal(0.0, 0.3, logits.shape)
        if round_bf16:
            ref = bf16_round(ref)
    return Case(logits=logits, token_ids=tok.astype(np.int32), seq_offsets=offs, advantages=adv,
                behavior_logp=behavior, row_of_token=rows, prox_logp=prox, engine_logp=eng, ref_logits=ref,
                rewards=rewards, group_offsets=go)


def config(variant: str, **kw) -> LossConfig:
    c = LossConfig(variant=LossVariant[variant], **{k: v for k, v in kw.items() if k != "aggregation"})
    if "aggregation" in kw:
        c.aggregation = RatioAggregation[kw["aggregation"]]
    return c


VARIANTS = ["ppo", "decoupled_ppo", "tis", "cispo", "topr", "grpo", "naive_is"]
