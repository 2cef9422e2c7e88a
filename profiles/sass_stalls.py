"""Warp-stall samples of an ncu --set full report, grouped by SASS opcode and by
contiguous code region (run here, no GPU):
    python profiles/sass_stalls.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys
from collections import Counter

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hi]
ai, si, ni = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
data = [r for r in rows[hi + 1:] if len(r) > ni and r[ai].startswith("0x")]
tot = sum(float(r[ni] or 0) for r in data)
ops, execd = Counter(), Counter()
for r in data:
    toks = r[si].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op] += float(r[ni] or 0)
    execd[op] += float(r[ei] or 0)
print(f"# {sys.argv[1]}: {tot:.0f} warp-stall samples")
print("## by opcode (share of samples, warp-instructions executed)")
for op, v in ops.most_common(30):
    print(f"{v / tot * 100:6.2f}%  {execd[op]:14.0f}  {op}")
print("## hottest instructions")
for r in sorted(data, key=lambda r: -float(r[ni] or 0))[:40]:
    print(f"{float(r[ni]) / tot * 100:6.2f}%  {r[ai]}  {r[si].strip()[:100]}")
