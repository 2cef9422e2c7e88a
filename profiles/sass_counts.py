"""Per-kernel SASS instruction counts of the shipped library (static, from
`cuobjdump -sass`), for the mnemonics that prove the Blackwell data paths:
UBLKCP / UTMALDG (TMA bulk / tensor copies), LDTM / STTM (tcgen05.ld/st, tensor
memory), UTCHMMA (tcgen05.mma), UTCBAR (tcgen05.commit), SYNCS (mbarrier ops),
MUFU.EX2, FFMA2 / FMUL2 / FADD2 (packed fp32), DSMEM remote stores (ST with
cluster addresses show as STS after MAPA), F2FP (packs), DADD/DMUL/DFMA (fp64).

    python profiles/sass_counts.py paper_2510_11345_b200/librf_offpolicy.so > profiles/r02_sass/sass_counts.txt
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "LDTM", "STTM", "UTCHMMA", "UTCBAR", "SYNCS", "MAPA", "MUFU.EX2",
        "FFMA2", "FMUL2", "FADD2", "HMNMX2", "F2FP", "DADD", "DMUL", "DFMA", "STG.E.128", "LDS.128", "STL", "LDL"]

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True, check=True).stdout
counts = defaultdict(Counter)
cur = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None or "/*" not in line:
        continue
    ins = line.split("*/", 1)[-1].strip().rstrip(";").strip()
    if not ins or ins.startswith("/*"):
        continue
    op = ins.split()[0]
    if op.startswith("@"):
        op = ins.split()[1]
    counts[cur]["total"] += 1
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            counts[cur][k] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


names = sorted(counts)
pretty = dict(zip(names, demangle(names)))
print(f"# cuobjdump -sass {sys.argv[1]}: static instruction counts per kernel")
for n in names:
    c = counts[n]
    fields = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
    print(f"{pretty[n][:90]:90s} total={c['total']} {fields}")
