"""Per-phase cycle breakdown of the fused kernel (run on the GPU box, profiling build):
    make -C paper_2510_11345_b200 phase
    RF_LIB_VARIANT=phase RF_DEBUG_COUNTERS=1 python tools/phase_profile.py [--prompts 32] [--kl]
Prints, per consumer warp, where the cycles of one launch of K2 (or, with --kl, of the
exact-KL kernel K2kl) went."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import _abi, synth as S  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402
from tests.cases import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prompts", type=int, default=32)
ap.add_argument("--variant", default="decoupled_ppo")
ap.add_argument("--kl", action="store_true", help="exact-KL GRPO (K2kl, 4-CTA groups)")
a = ap.parse_args()
assert os.environ.get("RF_DEBUG_COUNTERS") == "1"
wl = S.WORKLOADS["c2"]
rb = S.make_rank_batch(wl, 0, 1, 42, a.prompts)
dw = S.DeviceWorkload(rb, wl.vocab, pool_gb=8, device="cuda")
ref = None
if a.kl:
    ref = (torch.randn(dw.pool_rows, (wl.vocab + 7) // 8 * 8, device="cuda") * 2.0).to(torch.bfloat16)[:, :wl.vocab]
pb = L.PackedBatch(logits=dw.pool, token_ids=dw.token_ids, seq_offsets=dw.seq_offsets, advantages=dw.advantages,
                   behavior_logp=dw.behavior_logp, row_of_token=dw.row_of_token, prox_logp=dw.prox_logp,
                   engine_logp=dw.engine_logp, normalization=L.Normalization.global_token, ref_logits=ref)
cfg = config("grpo", kl_weight=0.1) if a.kl else config(a.variant)
op = rf.OffPolicyLoss(cfg, pb, chunk_tokens=min(65536, dw.T))
lib = _abi.load_library()
NCTA_MAX = 1024
buf = np.zeros(16 + 8 * NCTA_MAX, dtype=np.uint64)
for rep in range(3):
    op.zero()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    op.run(pb, 0, op.chunk)
    ev1.record()
    torch.cuda.synchronize()
    lib.rf_debug_counters(buf.ctypes.data, buf.size, 1)
ms = ev0.elapsed_time(ev1)
names = ["cons.full_wait", "cons.stream", "cons.park", "cons.coef_wait", "cons.write", "cons.total",
         "scal.red_wait", "scal.peer_wait", "scal.math", "scal.total", "prod.empty_wait", "prod.total",
         "scal.post_to_k", "scal.post.lse", "scal.post.token_post"]
if a.kl:  # K2kl: slot 12 = exchange done -> coefficient published, slot 13 = combining the warps' partials
    names[12:15] = ["scal.post_to_bcast", "scal.combine", "-"]
ncta = 148
bpt = (6 if a.kl else 4) * wl.vocab
print(f"launch {ms:.3f} ms for {op.chunk} tokens -> {op.chunk * bpt / ms / 1e6:.1f} GB/s ({'K2kl' if a.kl else 'K2'})")
cons_warps = ncta * 12
for i, n in enumerate(names):
    div = cons_warps if n.startswith("cons") else (ncta * 2 if n.startswith("scal") else ncta)
    print(f"{n:18s} {buf[i] / div / 1e3:10.1f} kcycles per warp   ({buf[i] / max(buf[5 if n.startswith('cons') else (9 if n.startswith('scal') else 11)], 1) * 100:5.1f}%)")
# per-CTA consumer spans of the last launch: how much of the launch is the tail (CTAs finishing early
# wait for the slowest group; static row assignment cannot rebalance)
tt = buf[16:].reshape(-1, 8).astype(np.int64)
tt = tt[(tt[:, 0] > 0) & (tt[:, 1] > 0)]
if len(tt):
    t0 = tt[:, 0].min()
    end = (tt[:, 1] - t0) / 1e3
    span = (tt[:, 1] - tt[:, 0]) / 1e3
    q = np.percentile(end, [0, 10, 50, 90, 100])
    print(f"CTA end times (us after the first CTA started), {len(tt)} CTAs: min {q[0]:.1f}  p10 {q[1]:.1f}  "
          f"median {q[2]:.1f}  p90 {q[3]:.1f}  max {q[4]:.1f};  mean {end.mean():.1f} -> tail {(q[4] - end.mean()) / q[4] * 100:.1f}% of the launch")
    print(f"CTA start skew: {(tt[:, 0].max() - t0) / 1e3:.1f} us; consumer spans: min {span.min():.1f}  max {span.max():.1f} us")
    order = np.argsort(tt[:, 2])
    tot = tt[:, 4:8].sum(axis=1).clip(min=1)
    print("per CTA by %smid (consumer warp 0): smid rows span_us us_per_row  full_wait% stream% coef_wait% write%")
    for i in order:
        f = tt[i, 4:8] / tot[i] * 100
        print(f"  {tt[i, 2]:4d} {tt[i, 3]:5d} {span[i]:9.1f} {span[i] / max(tt[i, 3], 1):7.3f}   "
              f"{f[0]:5.1f} {f[1]:5.1f} {f[2]:5.1f} {f[3]:5.1f}")
