"""Executed warp instructions per source line (all opcodes), top N, with the opcode mix of each:
python tools/ncu_lineinst.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None
cur = None
f = "?"
agg = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        ei = h.index("Instructions Executed")
        continue
    if h is None or len(r) <= ei:
        continue
    if r[0]:
        cur = (f, int(r[0]))
        src[cur] = r[1].strip()[:70]
        continue
    op = r[3].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    try:
        n = int(r[ei] or 0)
    except ValueError:
        continue
    agg[cur][o.split(".")[0]] += n
tot = sum(sum(c.values()) for c in agg.values())
lst = sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]
for k, c in lst:
    n = sum(c.values())
    mix = " ".join(f"{o}:{v * 100 // n}" for o, v in c.most_common(4))
    print(f"{n / tot * 100:5.1f}% {k[0][:12]}:{k[1]:>4} {src.get(k, ''):70s} {mix}")
