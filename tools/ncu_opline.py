"""Which source lines execute a given SASS opcode (executed warp instructions):
python tools/ncu_opline.py report.ncu-rep OPCODE [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = None
cur = None
f = "?"
agg = collections.Counter()
src = {}
allop = 0
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
        cur = (f, r[0])
        src[cur] = r[1].strip()[:80]
        continue
    op = r[3].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    try:
        n = int(r[ei] or 0)
    except ValueError:
        continue
    if o.split(".")[0] == want:
        agg[cur] += n
        allop += n
for k, n in agg.most_common(top):
    print(f"{n / allop * 100:5.1f}% {k[0][:14]}:{k[1]:>4} {src.get(k, '')}")
