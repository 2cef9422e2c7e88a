"""Synthetic long-tail rollout batches of the BASELINE.json configs (setup, never timed).

Seeding follows the reference's own random-stream discipline so the batch
shapes are reproducible from its code: ``RngStream`` = mt19937_64 seeded with
splitmix ``mix64(seed, FNV-1a(name))`` (reference proj/include/rlsim/rng.hpp:
17-84, proj/src/rng.cpp:7-21).  Lengths are
``ceil(sample_latency(make_lognormal(ln(max_len/32), 1.2, max_len)))``
(latency.cpp:47-55,105-132); rewards are Bernoulli(p_prompt), p_prompt ~ U(0,1)
per prompt (scheduler.cpp:36-41); staleness s ~ U{0..alpha} per sequence.
Logits (N(0, 2^2) rounded to bf16), sampled tokens and the behaviour / proximal
/ engine log-probs are generated on the GPU from a seeded torch generator.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

M64 = (1 << 64) - 1


def mix64(*args: int) -> int:
    """splitmix64 finalizer and its 2/3-argument chains (rng.hpp:17-31)."""

    def f(x: int) -> int:
        x = (x + 0x9E3779B97F4A7C15) & M64
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
        return x ^ (x >> 31)

    if len(args) == 1:
        return f(args[0])
    if len(args) == 2:
        return f(f(args[0]) ^ args[1])
    return f(mix64(args[0], args[1]) ^ args[2])


def stream_id(name: str) -> int:
    """FNV-1a (rng.hpp:33-40)."""
    h = 0xCBF29CE484222325
    for ch in name.encode():
        h ^= ch
        h = (h * 0x100000001B3) & M64
    return h


class MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & M64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M64


class RngStream:
    """rlsim::RngStream (rng.hpp:44-84, rng.cpp:7-21)."""

    def __init__(self, seed: int, stream):
        self.seed = seed
        self.stream = stream_id(stream) if isinstance(stream, str) else int(stream)
        self.gen = MT19937_64(mix64(seed, self.stream))

    def substream(self, name_or_idx, idx: Optional[int] = None) -> "RngStream":
        if idx is None:
            return RngStream(self.seed, mix64(self.stream, int(name_or_idx)))
        return RngStream(self.seed, mix64(self.stream, stream_id(name_or_idx), int(idx)))

    def next_u64(self) -> int:
        return self.gen()

    def uniform01(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def uniform01_open_low(self) -> float:
        return ((self.next_u64() >> 11) + 1.0) * 2.0 ** -53

    def normal(self, mean: float = 0.0, stddev: float = 1.0) -> float:
        u1 = self.uniform01_open_low()
        u2 = self.uniform01()
        z = math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)
        return mean + stddev * z

    def bernoulli(self, p: float) -> bool:
        return self.uniform01() < p

    def below(self, n: int) -> int:
        if n == 0:
            return 0
        limit = M64 - M64 % n
        x = self.next_u64()
        while x >= limit:
            x = self.next_u64()
        return x % n


def sample_lognormal_bounded(rng: RngStream, log_mean: float, log_std: float, upper: float) -> float:
    """sample_latency for a lognormal model: rejection to [0, upper], 100 tries, then clamp (latency.cpp:105-132)."""
    if log_std == 0.0:
        return min(max(math.exp(log_mean), 0.0), upper)
    v = 0.0
    for _ in range(100):
        v = math.exp(rng.normal(log_mean, log_std))
        if 0.0 <= v <= upper:
            return v
    return min(max(v, 0.0), upper)


# ---------------------------------------------------------------------------
# Workload configs (BASELINE.json "configs")
# ---------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    variant: str
    prompts: int
    group: int
    vocab: int
    max_len: int
    alpha: int
    description: str


WORKLOADS = {
    "c1": Workload("c1", "ppo", 64, 8, 32000, 1024, 1,
                   "GRPO + PPO-clip, 64 prompts x 8 responses, vocab 32k, max len 1k, long-tail lengths"),
    "c2": Workload("c2", "decoupled_ppo", 256, 8, 151936, 8192, 2,
                   "Qwen3-8B vocab (151936) decoupled-PPO loss+dlogits, 256 prompts x 8 responses, max len 8k, "
                   "async ratio 2"),
    "c3": Workload("c3", "tis", 512, 16, 151936, 16384, 2,
                   "TIS (and TOPR) off-policy variants, Qwen3 vocab, 512x16 responses, lognormal long-tail up to 16k"),
    "c4": Workload("c4", "cispo", 1024, 8, 151936, 32768, 8,
                   "CISPO loss with async ratio 8, Qwen3 vocab, 1024x8 responses, max len 32k"),
    "c5": Workload("c5", "decoupled_ppo", 2048, 16, 151936, 32768, 2,
                   "full box sweep: Qwen3 vocab, 2048 prompts x 16 responses, max len 32k, sequence-sharded"),
}


def sequence_lengths(seed: int, n: int, max_len: int, sigma: float = 1.2) -> np.ndarray:
    rng = RngStream(seed, "lengths")
    mu = math.log(max_len / 32.0)
    out = np.empty(n, dtype=np.int64)
    for i in range(n):
        out[i] = max(1, int(math.ceil(sample_lognormal_bounded(rng, mu, sigma, float(max_len)))))
    return out


def group_rewards(seed: int, prompts: int, group: int) -> np.ndarray:
    """Bernoulli(p_prompt) per response, p_prompt ~ U(0,1) (scheduler.cpp:36-41 semantics)."""
    root = RngStream(seed, "rewards")
    out = np.empty(prompts * group, dtype=np.float64)
    for p in range(prompts):
        pr = root.substream("difficulty", p).uniform01()
        for r in range(group):
            out[p * group + r] = 1.0 if root.substream("reward-value", mix64(p, r)).bernoulli(pr) else 0.0
    return out


def staleness(seed: int, n: int, alpha: int) -> np.ndarray:
    rng = RngStream(seed, "staleness")
    return np.array([rng.below(alpha + 1) for _ in range(n)], dtype=np.int64)


from .dist import lpt_shard  # noqa: E402  (whole-group LPT sharding)


@dataclass
class RankBatch:
    """Host-side description of one rank's shard (whole groups)."""

    lengths: np.ndarray      # [N_r]
    rewards: np.ndarray      # [N_r]
    stale: np.ndarray        # [N_r]
    group: int
    global_tokens: int
    global_seqs: int

    @property
    def num_tokens(self) -> int:
        return int(self.lengths.sum())


def make_rank_batch(wl: Workload, rank: int, world: int, seed: int = 42, prompts_per_rank: Optional[int] = None,
                    strong: bool = False):
    """This rank's shard (whole groups, LPT on group token counts) of the global batch.

    strong=False (weak scaling): global batch = world x (prompts per rank) prompts.
    strong=True (strong scaling): the config's fixed global batch (``prompts_per_rank``
    overrides the global prompt count) sharded over the world — the C5 sweep
    (BASELINE.json configs[4], "batch evaluation may be data-parallel")."""
    P = (prompts_per_rank or wl.prompts) * (1 if strong else world)
    G = wl.group
    lens = sequence_lengths(seed, P * G, wl.max_len)
    rew = group_rewards(seed, P, G)
    st = staleness(seed, P * G, wl.alpha)
    gt = lens.reshape(P, G).sum(axis=1)
    mine = lpt_shard(gt, world)[rank]
    if not mine:
        raise ValueError(f"rank {rank} of {world} owns no GRPO group ({P} groups)")
    idx = np.concatenate([np.arange(g * G, (g + 1) * G) for g in mine])
    return RankBatch(lengths=lens[idx], rewards=rew[idx], stale=st[idx], group=G,
                     global_tokens=int(lens.sum()), global_seqs=P * G)


class DeviceWorkload:
    """Device tensors for one rank: a logits pool (rows reused by token index
    modulo the pool size, so every read is a real HBM read), tokens drawn from
    each pool row's softmax, and behaviour/prox/engine log-probs staled as in
    BASELINE.md §4."""

    def __init__(self, rb: RankBatch, vocab: int, *, pool_gb: float = 48.0, device="cuda", seed: int = 42,
                 draws_per_row: int = 16):
        dev = torch.device(device)
        self.vocab = V = vocab
        T = rb.num_tokens
        N = len(rb.lengths)
        row_bytes = V * 2
        pool_rows = int(min(max(pool_gb * 1e9 // row_bytes, 1), T))
        self.pool_rows = pool_rows
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        padV = (V + 7) // 8 * 8
        pool = torch.empty(pool_rows, padV, dtype=torch.bfloat16, device=dev)
        step = max(1, int(2e9 // (padV * 4)))
        for r0 in range(0, pool_rows, step):
            r1 = min(pool_rows, r0 + step)
            pool[r0:r1].copy_(torch.randn(r1 - r0, padV, generator=gen, device=dev) * 2.0)
        self.pool = pool[:, :V]
        # per-row lse (fp64) and draws_per_row sampled tokens per row
        lse = torch.empty(pool_rows, dtype=torch.float64, device=dev)
        draws = torch.empty(pool_rows, draws_per_row, dtype=torch.int64, device=dev)
        step = max(1, int(2e9 // (V * 8)))
        for r0 in range(0, pool_rows, step):
            r1 = min(pool_rows, r0 + step)
            x = self.pool[r0:r1].double()
            lse[r0:r1] = torch.logsumexp(x, dim=1)
            p = torch.softmax(x.float(), dim=1)
            draws[r0:r1] = torch.multinomial(p, draws_per_row, replacement=True, generator=gen)
            del x, p
        t = torch.arange(T, device=dev, dtype=torch.int64)
        rows = t % pool_rows
        k = (t // pool_rows) % draws_per_row
        tok = draws[rows, k]
        lp = self.pool[rows, tok].double() - lse[rows]
        lens = torch.from_numpy(rb.lengths).to(dev)
        s_tok = torch.repeat_interleave(torch.from_numpy(rb.stale).to(dev).double(), lens)
        delta = torch.randn(T, generator=gen, device=dev, dtype=torch.float64) * 0.05 * torch.sqrt(s_tok)
        self.row_of_token = rows.to(torch.int32)
        self.token_ids = tok.to(torch.int32)
        self.lp_theta = lp
        self.behavior_logp = (lp - delta).to(torch.float32)
        self.prox_logp = (lp - 0.5 * delta).to(torch.float32)
        self.engine_logp = (self.behavior_logp.double() -
                            0.01 * torch.randn(T, generator=gen, device=dev, dtype=torch.float64)).to(torch.float32)
        offs = torch.zeros(N + 1, dtype=torch.int64)
        offs[1:] = torch.cumsum(torch.from_numpy(rb.lengths), 0)
        self.seq_offsets = offs.to(dev)
        self.rewards = torch.from_numpy(rb.rewards).to(dev)
        G = rb.group
        self.group_offsets = (torch.arange(N // G + 1, dtype=torch.int64) * G).to(dev)
        self.advantages = torch.zeros(N, dtype=torch.float64, device=dev)
        self.T = T
        self.N = N
        self.rb = rb
