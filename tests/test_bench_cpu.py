"""CPU: bench.py's reference arm and its process hygiene.

The driver's reference arm (``bench.py --impl reference``) must time the
reference's own CPU implementation (oracle/_ref, compiled from /root/reference)
and must NOT map the product library librf_offpolicy.so.
"""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WRAP = r"""
import runpy, sys, json
sys.argv = ["bench.py", "--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0",
            "--cpu-rows", "16"]
try:
    runpy.run_path({bench!r}, run_name="__main__")
finally:
    maps = sorted({{l.split()[-1] for l in open("/proc/self/maps") if l.rstrip().endswith(".so")}})
    print("MAPS " + json.dumps(maps))
"""


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_does_not_map_product_library():
    r = subprocess.run([sys.executable, "-c", _WRAP.format(bench=os.path.join(ROOT, "bench.py"))], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    line = json.loads(next(x for x in lines if x.startswith("{")))
    maps = json.loads(next(x for x in lines if x.startswith("MAPS "))[5:])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert any(m.endswith("oracle/_ref/librlsim_ref.so") for m in maps), maps
    assert not any("librf_offpolicy" in m for m in maps), maps


def test_strong_scaling_shards_the_fixed_global_batch():
    from paper_2510_11345_b200 import synth as S

    wl = S.WORKLOADS["c1"]
    one = S.make_rank_batch(wl, 0, 1, 42, strong=True)
    parts = [S.make_rank_batch(wl, r, 4, 42, strong=True) for r in range(4)]
    assert sum(p.num_tokens for p in parts) == one.num_tokens == one.global_tokens
    assert all(p.global_tokens == one.global_tokens and p.global_seqs == one.global_seqs for p in parts)
    assert all(len(p.lengths) % wl.group == 0 for p in parts)
    # weak scaling: every rank a config-sized shard of an N x batch
    weak = S.make_rank_batch(wl, 0, 4, 42, strong=False)
    assert weak.global_seqs == 4 * one.global_seqs
