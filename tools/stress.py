"""Repeated launches of the fused kernel with per-launch sync and a watchdog
(hang / race hunting on the GPU box):
    timeout 300 python tools/stress.py --launches 200 [--prompts 256]"""
import argparse
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402
from paper_2510_11345_b200 import synth as S  # noqa: E402
from tests.cases import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prompts", type=int, default=64)
ap.add_argument("--launches", type=int, default=200)
ap.add_argument("--variant", default="decoupled_ppo")
ap.add_argument("--chunk", type=int, default=65536)
ap.add_argument("--pool-gb", type=float, default=8)
ap.add_argument("--random", action="store_true", help="random token ranges (1..chunk tokens) per launch")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--kl", action="store_true", help="exact-KL GRPO (a reference-policy pool row per token)")
a = ap.parse_args()
wl = S.WORKLOADS["c2"]
rb = S.make_rank_batch(wl, 0, 1, 42, a.prompts)
dw = S.DeviceWorkload(rb, wl.vocab, pool_gb=a.pool_gb, device="cuda")
ref = None
if a.kl:
    padV = (wl.vocab + 7) // 8 * 8
    ref = (torch.randn(dw.pool_rows, padV, device="cuda") * 2.0).to(torch.bfloat16)[:, : wl.vocab]
pb = L.PackedBatch(logits=dw.pool, token_ids=dw.token_ids, seq_offsets=dw.seq_offsets, advantages=dw.advantages,
                   behavior_logp=dw.behavior_logp, row_of_token=dw.row_of_token, prox_logp=dw.prox_logp,
                   engine_logp=dw.engine_logp, normalization=L.Normalization.global_token, ref_logits=ref)
chunk = min(a.chunk, dw.T)
cfg = config("grpo", kl_weight=0.1) if a.kl else (L.LossConfig() if a.variant == "ppo" else config(a.variant))
op = rf.OffPolicyLoss(cfg, pb, chunk_tokens=chunk)
last = [time.time(), 0]
done = [False]


def watchdog():
    while not done[0]:
        time.sleep(1.0)
        if time.time() - last[0] > 15:
            print(f"WATCHDOG: launch {last[1]} not finished after 15 s", flush=True)
            last[0] = time.time()


threading.Thread(target=watchdog, daemon=True).start()
ref = None
chunks = [(t0, min(dw.T, t0 + chunk)) for t0 in range(0, dw.T, chunk)]
t_start = time.time()
import random  # noqa: E402

rng = random.Random(a.seed)
probe = (0, min(dw.T, 4096))  # re-run periodically: outputs must be bit-identical (race check)
probe_sig = None
for i in range(a.launches):
    if a.random:
        n = rng.randint(1, chunk)
        t0 = rng.randint(0, dw.T - n)
        t0, t1 = t0, t0 + n
    else:
        t0, t1 = chunks[i % len(chunks)]
    if i % 25 == 0:
        t0, t1 = probe
    op.zero()
    op.run(pb, t0, t1)
    torch.cuda.synchronize()
    last[0] = time.time()
    last[1] = i
    if (t0, t1) == probe:
        sig = (op.scalars.clone().cpu(), op.dlogits[: t1 - t0].float().sum(dim=1).cpu())
        if probe_sig is None:
            probe_sig = sig
        elif not (torch.equal(sig[0], probe_sig[0]) and torch.equal(sig[1], probe_sig[1])):
            print(f"MISMATCH at launch {i}: probe outputs differ from the first run", flush=True)
            sys.exit(2)
    if int(op.status.item()) != 0:
        print(f"device status {int(op.status.item())} at launch {i} ({t0}, {t1})", flush=True)
        sys.exit(3)
    if (i + 1) % 100 == 0:
        print(f"launch {i + 1} ok ({time.time() - t_start:.1f} s)", flush=True)
done[0] = True
print("stress done", flush=True)
