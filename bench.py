#!/usr/bin/env python
"""Benchmark: fused off-policy loss + dlogits tokens/s and % HBM roofline on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl ours|reference]

One step = the hot path over one synthetic long-tail rollout batch of a
BASELINE.json config.  Default: C5, the config the metric's 1/2/4/8-GPU sweep is
quoted on (Qwen3 vocab 151,936, 2048 prompts x 16 responses, max len 32k,
decoupled PPO, async ratio 2), a FIXED global batch whose whole GRPO groups are
LPT-sharded over the ranks (strong scaling; ``--scaling weak`` gives every rank
its own copy-sized shard instead):
  K1 GRPO group advantages -> K2 fused log-softmax/gather + ratio + surrogate +
  bf16 dlogits, streamed in token chunks from a device logits pool (rows indexed
  by row_of_token; pool and dlogits buffers far exceed L2) -> K3 scalar reduce ->
  (N > 1) one NCCL all-reduce of the fp64 loss scalars.
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  ``--gpus N`` without a torchrun environment re-launches
itself under torch.distributed.run with N ranks.

After the timed region: ``e2e`` (the C-ABI host-buffer call, every rank at
once), ``cpu_baseline`` (rank 0, N = 1) and the ``--check K`` leg, which holds
K sampled token rows of the last timed step (plus every GRPO group's
advantages) to the fp64 oracle (oracle/check.py) — checkers, never timed.

--impl reference times the reference's own CPU implementation (rlsim::loss_and_grad
compiled from /root/reference into oracle/_ref, one length-1 trajectory per token)
on the host cores, rank 0 only; that arm never maps the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "loss+dlogits tokens/sec and % HBM roofline at 1/2/4/8 B200 vs CPU ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's fixed global batch sharded over N; weak: N copies")
    ap.add_argument("--variant", default=None)
    ap.add_argument("--aggregation", default="token_mean", choices=["token_mean", "sequence_product"])
    ap.add_argument("--prompts", type=int, default=None,
                    help="prompts (global for strong scaling, per rank for weak; default: the config's)")
    ap.add_argument("--chunk-tokens", type=int, default=65536)
    ap.add_argument("--pool-gb", type=float, default=48.0)
    ap.add_argument("--kernel", default="auto", choices=["auto", "ring", "generic"])
    ap.add_argument("--kl-weight", type=float, default=0.0,
                    help="exact-KL GRPO (variant grpo, a reference-policy row per token, 6·V B/token)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-tokens", type=int, default=16384)
    ap.add_argument("--cpu-rows", type=int, default=0, help="reference sample rows (0 = auto)")
    ap.add_argument("--check", type=int, default=256,
                    help="oracle parity on this many sampled token rows of the last timed step (0 = off)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(n: int) -> None:
    """`python bench.py --gpus N` outside torchrun: re-exec with N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd[2:6])} ...", file=sys.stderr, flush=True)
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def static_traffic(key: str):
    """dram read+write bytes per token of the dominant kernel from a committed
    `ncu --set full` capture (profiles/ring_traffic.json) — a static file value,
    not measured in this run."""
    try:
        with open(os.path.join(ROOT, "profiles", "ring_traffic.json")) as f:
            d = json.load(f)
        e = d.get(key)
        return None if e is None else (e["dram_bytes_per_token"], e.get("source", ""))
    except Exception:
        return None


def make_config(variant: str, aggregation: str = "token_mean", kl_weight: float = 0.0):
    """rlsim::LossConfig defaults (losses.hpp:28-41) for the named variant."""
    from paper_2510_11345_b200.losses import LossConfig, LossVariant, RatioAggregation

    return LossConfig(variant=LossVariant[variant], aggregation=RatioAggregation[aggregation], kl_weight=kl_weight)


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref): rlsim::loss_and_grad on mapping-A rows
# ---------------------------------------------------------------------------
def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_sample(wl, rows, variant, seed=42):
    """A bounded, seeded sample of the same workload on the host: `rows` token rows
    (bf16 logits as fp64), tokens, advantages, behaviour/prox/engine log-probs."""
    import numpy as np

    from paper_2510_11345_b200 import synth as S  # host-side shapes only (no product library)

    rb = S.make_rank_batch(wl, 0, 1, seed)
    rng = np.random.default_rng(seed)
    V = wl.vocab
    x = rng.normal(0.0, 2.0, (rows, V)).astype(np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    x = (((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)).view(np.float32).astype(np.float64)
    m = x.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(x - m).sum(axis=1, keepdims=True)))[:, 0]
    tok = np.empty(rows, dtype=np.int32)
    for r0 in range(0, rows, 256):  # Gumbel-max sampling, chunked to bound host memory
        r1 = min(rows, r0 + 256)
        tok[r0:r1] = np.argmax(x[r0:r1] + rng.gumbel(size=(r1 - r0, V)), axis=1)
    lp = x[np.arange(rows), tok] - lse
    seq = np.repeat(np.arange(len(rb.lengths)), rb.lengths)[:rows]
    s = rb.stale[seq]
    delta = rng.normal(0.0, 1.0, rows) * 0.05 * np.sqrt(s)
    beh = lp - delta
    prox = lp - delta / 2
    eng = beh - rng.normal(0.0, 0.01, rows)
    adv = np.zeros(len(rb.lengths))
    G = rb.group
    for gi in range(len(rb.lengths) // G):
        r = rb.rewards[gi * G:(gi + 1) * G]
        mean = r.sum() / G
        sd = np.sqrt(((r - mean) ** 2).sum() / G)
        if sd >= 1e-8:
            adv[gi * G:(gi + 1) * G] = (r - mean) / sd
    return x, tok, adv[seq], beh, prox, eng


def prepare_reference(wl, variant, rows):
    """Sample + the prox ToyPolicy table the reference needs (setup, untimed)."""
    import oracle as O

    x, tok, adv, beh, prox, eng = reference_sample(wl, rows, variant)
    prox_tab = O.ref_build_prox_table(x, tok, prox) if variant == "decoupled_ppo" else None
    return (x, tok, adv, beh, prox_tab)


def run_reference_once(prep, cfg, threads, reps=1):
    """Wall seconds of rlsim::loss_and_grad over the prepared rows (oracle/_ref)."""
    import oracle as O

    x, tok, adv, beh, prox_tab = prep
    secs, _ = O.ref_bench_mapping_a(cfg, x, tok, adv, beh, prox_logits=prox_tab, engine_logp=None,
                                    threads=threads, reps=reps)
    return secs


def default_cpu_rows(wl, threads):
    per_core = 96 if wl.vocab > 100000 else 400
    return int(min(max(per_core * threads, 128), 2048 if wl.vocab > 100000 else 8192))


def cpu_baseline(wl, variant, rows):
    threads = host_threads()
    rows = rows or default_cpu_rows(wl, threads)
    secs = run_reference_once(prepare_reference(wl, variant, rows), make_config(variant), threads)
    return {"value": rows / secs, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": f"{rows} token rows of {wl.name} (V={wl.vocab}, {variant}, mapping A: one length-1 "
                      f"trajectory per token), rlsim::loss_and_grad from oracle/_ref on {threads} host threads "
                      f"(one shard each), {secs:.2f} s wall"}


def impl_reference(args, wl, variant):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = host_threads()
    rows = args.cpu_rows or default_cpu_rows(wl, threads)
    prep = prepare_reference(wl, variant, rows)
    cfg = make_config(variant)
    for _ in range(args.warmup):
        run_reference_once(prep, cfg, threads)
    times = [run_reference_once(prep, cfg, threads) for _ in range(args.steps)]
    mean = sum(times) / len(times)
    value = rows / mean
    sample = (f"{rows} token rows of {wl.name} per step (V={wl.vocab}, {variant}, mapping A), "
              f"rlsim::loss_and_grad from oracle/_ref on {threads} host threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.description, "variant": variant, "vocab": wl.vocab, "sample_rows": rows},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def e2e_host_api(cfg, dw, tokens, world, steps=3, warmup=1, chunk=512, ref_pool=None):
    """The reference-facing C-ABI call with HOST buffers (rf_loss_and_grad_host), on
    every rank at once: pinned host logits rows in, pinned host dlogits + per-token
    outputs + scalars out; every H2D/D2H copy is inside the timed region.  Returns the
    whole-job tokens/s (sum of the ranks' tokens / the slowest rank's step time)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2510_11345_b200 import _abi
    from paper_2510_11345_b200 import losses as L

    V = dw.vocab
    try:  # bound the pinned host memory (logits + dlogits rows) by the box's free RAM
        import psutil

        avail = psutil.virtual_memory().available
        tokens = int(max(512, min(tokens, avail * 0.25 / world / (4 * V))))
    except Exception:
        pass
    offs = dw.seq_offsets.cpu()
    n_seq = int(torch.searchsorted(offs, torch.tensor([min(tokens, dw.T)]), right=True)[0]) - 1
    n_seq = max(n_seq, 1)
    T = int(offs[n_seq])
    rows = dw.row_of_token[:T].long()
    h_logits = torch.empty(T, V, dtype=torch.bfloat16, pin_memory=True)
    for r0 in range(0, T, 4096):
        h_logits[r0:r0 + 4096].copy_(dw.pool[rows[r0:r0 + 4096]].cpu())
    h_dl = torch.empty(T, V, dtype=torch.bfloat16, pin_memory=True)
    h_ref = None
    if ref_pool is not None:  # exact KL: the reference-policy row of every token too
        h_ref = torch.empty(T, V, dtype=torch.bfloat16, pin_memory=True)
        for r0 in range(0, T, 4096):
            h_ref[r0:r0 + 4096].copy_(ref_pool[rows[r0:r0 + 4096]].cpu())

    def pin(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t.cpu())
        return h

    h_tok = pin(dw.token_ids[:T])
    h_seq = pin(L.seq_of_token_from_offsets(dw.seq_offsets[: n_seq + 1]))
    h_offs = pin(dw.seq_offsets[: n_seq + 1])
    h_adv = pin(dw.advantages[:n_seq])
    h_b = pin(dw.behavior_logp[:T])
    h_q = pin(dw.prox_logp[:T])
    h_e = pin(dw.engine_logp[:T])
    outs = {k: torch.empty(T, dtype=torch.float64, pin_memory=True) for k in ["lp", "ratio", "coef", "loss"]}
    h_flags = torch.empty(T, dtype=torch.uint8, pin_memory=True)
    h_scal = torch.zeros(_abi.RF_NUM_SCALARS, dtype=torch.float64, pin_memory=True)
    h_status = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    c = cfg.to_c()
    b = _abi.rf_batch()
    b.num_tokens, b.num_seqs, b.vocab = T, n_seq, V
    b.logits_dtype, b.logits, b.logits_row_stride = _abi.RF_DTYPE_BF16, h_logits.data_ptr(), V
    b.token_ids, b.seq_of_token, b.seq_offsets = h_tok.data_ptr(), h_seq.data_ptr(), h_offs.data_ptr()
    b.advantages = h_adv.data_ptr()
    b.logp_dtype, b.normalization = _abi.RF_DTYPE_F32, _abi.RF_NORM_GLOBAL_TOKEN
    b.behavior_logp, b.prox_logp, b.engine_logp = h_b.data_ptr(), h_q.data_ptr(), h_e.data_ptr()
    b.global_num_seqs, b.global_num_tokens, b.grad_sign = n_seq, T, 1.0
    if h_ref is not None:
        b.ref_logits, b.ref_row_stride = h_ref.data_ptr(), V
    o = _abi.rf_outputs()
    o.dlogits, o.dlogits_dtype, o.dlogits_row_stride = h_dl.data_ptr(), _abi.RF_DTYPE_BF16, V
    o.token_logp, o.token_ratio = outs["lp"].data_ptr(), outs["ratio"].data_ptr()
    o.token_coef, o.token_loss, o.token_flags = outs["coef"].data_ptr(), outs["loss"].data_ptr(), h_flags.data_ptr()
    o.scalars, o.device_status = h_scal.data_ptr(), h_status.data_ptr()
    lib = _abi.load_library()
    dev = torch.cuda.current_device()
    for _ in range(warmup):
        st = lib.rf_loss_and_grad_host(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), dev, chunk)
        assert st == 0, L.status_string(st)
    ts = []
    for _ in range(steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        st = lib.rf_loss_and_grad_host(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), dev, chunk)
        ts.append(time.perf_counter() - t0)
        assert st == 0, L.status_string(st)
    tt = torch.tensor(ts + [float(T)], dtype=torch.float64, device=f"cuda:{dev}")
    if world > 1:
        tsum = tt[-1:].clone()
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        T_all = int(tsum.item())
    else:
        T_all = T
    t = statistics.median(tt[:-1].tolist())
    h2d = T * V * 2 * (2 if h_ref is not None else 1) + T * (4 + 4 + 4 * 3) + (n_seq + 1) * 8 + n_seq * 8
    d2h = T * V * 2 + T * (8 * 4 + 1) + _abi.RF_NUM_SCALARS * 8 + 4
    return {"value": T_all / t, "unit": "tokens/s", "h2d_bytes_per_step": int(h2d * world),
            "d2h_bytes_per_step": int(d2h * world),
            "sample": f"first {T} tokens ({n_seq} whole sequences) of each rank's shard per step on {world} "
                      f"rank(s) at once, rf_loss_and_grad_host (C ABI, pinned host buffers, {chunk}-token chunks "
                      f"double-buffered over H2D/compute/D2H streams), median over {steps} steps of the slowest "
                      f"rank's wall-clock step"}


def parity_leg(K, cfg, dw, rb, op, calls, k1_out, ref_pool, rank, world, dev, seqprod):
    """Checker (not timed): K sampled token rows of the last timed step vs the fp64
    oracle, and every GRPO group's advantages bit-exact.  Returns the merged stats
    (max over ranks, ``ok`` = every rank ok)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    from oracle.check import check_sample

    rng = np.random.default_rng(4321 + rank)
    st, adv_o, deg_o = O.oracle_grpo(dw.rewards.cpu().numpy(), dw.group_offsets.cpu().numpy())
    k1_ok = st == 0 and np.array_equal(k1_out[0].cpu().numpy(), adv_o) and \
        np.array_equal(k1_out[1].cpu().numpy(), deg_o)
    _, t1_last, sub_last, out_t0 = calls[-1]
    t0_last = calls[-1][0]
    n_last = t1_last - t0_last
    offs = dw.seq_offsets.cpu().numpy()
    if not seqprod:
        a = rng.choice(n_last, size=min(K // 2, n_last), replace=False) + out_t0
        bsel = rng.choice(dw.T, size=max(0, K - len(a)), replace=False)
        toks = np.unique(np.concatenate([a, bsel]).astype(np.int64))
        sub_offs = np.arange(len(toks) + 1, dtype=np.int64)
        seq_ids = np.searchsorted(offs, toks, side="right") - 1
    else:
        # whole (short) sequences: half from the last call (their dlogits rows are still on the device)
        lens = np.diff(offs)
        s_last = np.nonzero((offs[:-1] >= out_t0) & (offs[1:] <= out_t0 + n_last) & (lens <= K // 4))[0]
        s_any = np.nonzero(lens <= K // 4)[0]
        pick, tot = [], 0
        for cand, cap in ((s_last, K // 2), (s_any, K)):
            for s in rng.permutation(cand):
                if tot >= cap:
                    break
                if int(s) not in pick:
                    pick.append(int(s))
                    tot += int(lens[s])
        pick = sorted(set(pick))
        toks = np.concatenate([np.arange(offs[s], offs[s + 1]) for s in pick]).astype(np.int64)
        sub_offs = np.zeros(len(pick) + 1, dtype=np.int64)
        sub_offs[1:] = np.cumsum(lens[pick])
        seq_ids = np.array(pick, dtype=np.int64)
    it = torch.from_numpy(toks).to(dev)
    rows = dw.row_of_token[it].long()
    X = dw.pool[rows].double().cpu().numpy()
    Y = ref_pool[rows].double().cpu().numpy() if ref_pool is not None else None
    f64 = lambda t: t[it].double().cpu().numpy()
    gpu = {"lp": f64(op.token_logp), "ratio": f64(op.token_ratio), "coef": f64(op.token_coef),
           "loss": f64(op.token_loss), "flags": op.token_flags[it].cpu().numpy()}
    dl = {}
    for i, t in enumerate(toks):
        if out_t0 <= t < out_t0 + n_last:
            dl[i] = op.dlogits[int(t - out_t0)].double().cpu().numpy()
    stats = check_sample(cfg, logits=X, token_ids=dw.token_ids[it].cpu().numpy(), seq_offsets=sub_offs,
                         advantages=k1_out[0][torch.from_numpy(seq_ids).to(dev)].cpu().numpy(),
                         behavior_logp=f64(dw.behavior_logp), prox_logp=f64(dw.prox_logp),
                         engine_logp=f64(dw.engine_logp), ref_logits=Y, normalization=1,
                         global_num_seqs=rb.global_seqs, global_num_tokens=rb.global_tokens, gpu=gpu, dl_rows=dl)
    stats["k1_groups_bit_exact"] = bool(k1_ok)
    stats["ok"] = bool(stats["ok"] and k1_ok)
    keys = ["lp_rel", "ratio_rel", "coef_rel", "token_loss_err", "dlogit_unit_err"]
    cnt = ["tokens", "dlogit_rows", "kink_band_tokens", "flag_mismatch", "flag_mismatch_in_band"]
    if world > 1:
        mx = torch.tensor([stats[k] for k in keys] + [0.0 if stats["ok"] else 1.0], dtype=torch.float64, device=dev)
        sm = torch.tensor([stats[k] for k in cnt] + [len(deg_o)], dtype=torch.float64, device=dev)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        stats.update({k: float(v) for k, v in zip(keys, mx.tolist()[:-1])})
        stats.update({k: int(v) for k, v in zip(cnt, sm.tolist()[:-1])})
        stats["ok"] = mx[-1].item() == 0.0
        stats["k1_groups"] = int(sm[-1].item())
    else:
        stats["k1_groups"] = len(deg_o)
    stats["checker"] = ("oracle/rf_oracle.c (fp64 restatement of losses.cpp:137-331, pinned to oracle/_ref) on "
                        "sampled rows of the last timed step; tolerances BASELINE.md §5")
    return stats


def impl_ours(args, wl, variant):
    import torch
    import torch.distributed as dist

    import paper_2510_11345_b200 as rf
    from paper_2510_11345_b200 import losses as L
    from paper_2510_11345_b200 import synth as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    strong = args.scaling == "strong"
    rb = S.make_rank_batch(wl, rank, world, 42, args.prompts, strong=strong)
    dw = S.DeviceWorkload(rb, wl.vocab, pool_gb=args.pool_gb, device=dev, seed=42 + rank)
    cfg = make_config(variant, args.aggregation, args.kl_weight)
    ref_pool = None
    if args.kl_weight > 0:
        # exact-KL GRPO: a second, independent pool of reference-policy rows (π_ref),
        # indexed by the same row_of_token, so every token reads both rows from HBM
        gen = torch.Generator(device=dev)
        gen.manual_seed(4242 + rank)
        full = torch.empty(dw.pool_rows, (wl.vocab + 7) // 8 * 8, dtype=torch.bfloat16, device=dev)
        step = max(1, int(2e9 // (full.shape[1] * 4)))
        for r0 in range(0, dw.pool_rows, step):
            r1 = min(dw.pool_rows, r0 + step)
            full[r0:r1].copy_(torch.randn(r1 - r0, full.shape[1], generator=gen, device=dev) * 2.0)
        ref_pool = full[:, : wl.vocab]
    pb = L.PackedBatch(logits=dw.pool, token_ids=dw.token_ids, seq_offsets=dw.seq_offsets, ref_logits=ref_pool,
                       advantages=dw.advantages, behavior_logp=dw.behavior_logp, row_of_token=dw.row_of_token,
                       prox_logp=dw.prox_logp, engine_logp=dw.engine_logp, rewards=dw.rewards,
                       group_offsets=dw.group_offsets, normalization=L.Normalization.global_token,
                       global_num_seqs=rb.global_seqs, global_num_tokens=rb.global_tokens)
    chunk = min(args.chunk_tokens, dw.T)
    stream = torch.cuda.current_stream()
    rf.grpo_advantages(pb.rewards, pb.group_offsets, stream)  # validates the group layout once
    k1_out = (torch.empty_like(pb.rewards), torch.empty(dw.group_offsets.numel() - 1, dtype=torch.uint8, device=dev),
              torch.zeros(1, dtype=torch.int32, device=dev))
    pb.advantages = k1_out[0]
    seqprod = args.aggregation == "sequence_product"
    if seqprod:
        # whole sequences per call (the sequence weights need every token's log-prob)
        calls = [(0, t1 - t0, sub, t0) for t0, t1, sub in pb.sequence_chunks(chunk)]
        chunk = max(c[1] for c in calls)
    else:
        calls = [(t0, min(dw.T, t0 + chunk), pb, t0) for t0 in range(0, dw.T, chunk)]
    op = rf.OffPolicyLoss(cfg, pb, chunk_tokens=chunk, kernel=args.kernel)
    # one event pair per (timed step, chunk): the kernel time is averaged over every timed step
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in calls]
          for _ in range(args.steps)]

    def step(record=None):
        rf.grpo_advantages(pb.rewards, pb.group_offsets, stream, out=k1_out, validate=False)
        op.zero(stream)
        for i, (t0, t1, b, out_t0) in enumerate(calls):
            if record is not None:
                ev[record][i][0].record(stream)
            op.run(b, t0, t1, stream, out_t0=out_t0)
            if record is not None:
                ev[record][i][1].record(stream)
        if world > 1:
            dist.all_reduce(op.scalars)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness guard on the benchmark data: device status clean
    assert int(op.status.item()) == 0 and int(k1_out[2].item()) == 0, "device status set during warm-up"
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern_ms = 0.0
    launches_before = op.launches
    start.record(stream)
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ selects exactly these launches
    for k in range(args.steps):
        step(record=k)
    torch.cuda.nvtx.range_pop()
    stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_total = start.elapsed_time(stop)
    # dominant-kernel time per step: every chunk's launch pair, averaged over the timed steps
    for evs in ev:
        for a, b2 in evs:
            kern_ms += a.elapsed_time(b2)
    kern_ms /= args.steps
    launches = (op.launches - launches_before) + args.steps  # + one K1 per step
    t_local = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step = float(t_local[0]) / args.steps
    tokens_global = rb.global_tokens  # the whole job: every rank's tokens
    value = tokens_global / (ms_step / 1e3)
    step_status = int(op.status.item())

    peak, peak_kind = load_peaks()
    kl = args.kl_weight > 0
    # token_mean: one read + one write of each row (4V B/token); sequence_product: a
    # stats read pass + a read/write dlogits pass (6V B/token); exact KL: + the π_ref row read
    bytes_tok = (6 if (seqprod or kl) else 4) * wl.vocab
    achieved = dw.T * bytes_tok / (kern_ms / 1e3) / 1e9
    tkey = ("seqprod" if seqprod else "kl" if kl else "lag") + f"/{wl.vocab}"
    tr = static_traffic(tkey)
    launch_tokens = calls[0][1] - calls[0][0]
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None if tr is None else int(tr[0] * launch_tokens),
            "traffic_source": None if tr is None else
            f"static: dram__bytes_read+write per token from a committed ncu --set full capture ({tr[1]}) x "
            f"{launch_tokens} tokens per launch; not measured in this run",
            "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, torch bf16 copy)" if peak_kind == "measured"
            else "fallback 6.65 TB/s (B200_PROFILING.md)",
            "kernel": ("stream_stats_kernel + seq_kernel + stream_write_kernel (+K3)" if seqprod
                       else "ring_kl_kernel (K2kl, incl. its K3 finalize launch)" if kl
                       else "ring_lag_kernel (K2, incl. its K3 finalize launch)"),
            "algorithmic_bytes_per_token": bytes_tok, "tokens_per_launch": launch_tokens,
            "kernel_ms_per_step": round(kern_ms, 3), "per_rank": True}

    # ---- after the timed region: e2e (all ranks), parity checker, CPU baseline ----
    e2e = None
    if not args.no_e2e:
        try:
            e2e = e2e_host_api(cfg, dw, args.e2e_tokens if world == 1 else min(args.e2e_tokens, 8192), world,
                               ref_pool=ref_pool)
        except Exception as exc:  # report, do not hide
            e2e = {"value": None, "unit": "tokens/s", "error": repr(exc)}
    parity = None
    if args.check > 0:
        try:
            parity = parity_leg(args.check, cfg, dw, rb, op, calls, k1_out, ref_pool, rank, world, dev, seqprod)
        except Exception as exc:
            parity = {"ok": False, "error": repr(exc)}
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(wl, variant, args.cpu_rows)
            except Exception as exc:
                cpu = {"value": None, "error": repr(exc)}
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl.description, "variant": variant, "aggregation": args.aggregation,
                       "kl_weight": args.kl_weight, "vocab": wl.vocab,
                       "prompts_global": (args.prompts or wl.prompts) * (1 if strong else world),
                       "group": wl.group, "max_len": wl.max_len, "async_ratio": wl.alpha,
                       "tokens_rank0": dw.T, "tokens_global": tokens_global,
                       "chunk_tokens": chunk, "logits_pool_rows": dw.pool_rows,
                       "l2": f"inputs larger than L2: logits pool {dw.pool_rows * wl.vocab * 2 / 1e9:.1f} GB, "
                             f"dlogits chunk buffer {chunk * wl.vocab * 2 / 1e9:.1f} GB (L2 126 MB)",
                       "accumulation": "fp32 softmax sums, fp64 per-token scalars and loss",
                       "parallelism": f"dp{world} (whole GRPO groups LPT-sharded, one fp64 NCCL all-reduce)",
                       "kernel": args.kernel},
            "roofline": roof,
            "clocks": clk,
            "gpu_launches": int(launches),
            "device_status": step_status,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    from paper_2510_11345_b200 import synth as S

    wl = S.WORKLOADS[args.workload]
    variant = args.variant or ("grpo" if args.kl_weight > 0 else wl.variant)
    if args.impl == "reference":
        impl_reference(args, wl, variant)
    else:
        impl_ours(args, wl, variant)


if __name__ == "__main__":
    main()
