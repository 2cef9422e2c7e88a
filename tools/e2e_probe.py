"""Probe the host-buffer C-ABI path (rf_loss_and_grad_host) on the GPU box:
per-call wall time at a few chunk sizes, next to the raw pinned H2D / D2H
bandwidth of the same bytes."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_11345_b200 import synth as S  # noqa: E402

wl = S.WORKLOADS["c2"]
rb = S.make_rank_batch(wl, 0, 1, 42, int(os.environ.get("E2E_PROMPTS", "16")))
dw = S.DeviceWorkload(rb, wl.vocab, pool_gb=4, device="cuda")
dw.advantages.fill_(0.5)
nbytes = 8192 * wl.vocab * 2
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s", flush=True)
# both directions at once (what the pipelined host call needs)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"h2d+d2h concurrent: {nbytes / dt / 1e9:.1f} GB/s per direction", flush=True)
chunks = [int(c) for c in os.environ.get("E2E_CHUNKS", "256,512,1024,2048").split(",")]
ntok = int(os.environ.get("E2E_TOKENS", "8192"))
for chunk in chunks:
    import ctypes  # noqa: F401

    r = bench.e2e_host_api.__wrapped__ if hasattr(bench.e2e_host_api, "__wrapped__") else bench.e2e_host_api
    t = time.perf_counter()
    out = r(wl, wl.variant, dw, ntok, steps=3, warmup=1, chunk=chunk)
    print(f"chunk {chunk}: e2e {out['value']:.0f} tok/s  (probe wall {time.perf_counter() - t:.1f} s)", flush=True)
