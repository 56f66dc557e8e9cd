"""SASS opcode mix (executed warp instructions) of an ncu report's source page:
python tools/ncu_opmix.py report.ncu-rep [n_dofs]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si, ei = h.index("Source"), h.index("Instructions Executed")
ndof = float(sys.argv[2]) if len(sys.argv) > 2 else 16974593
c = collections.Counter()
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= ei:
        continue
    try:
        n = int(r[ei] or 0)
    except ValueError:
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    c[o.split(".")[0]] += n
    tot += n
print(f"total warp instructions {tot}, {tot * 32 / ndof:.1f} thread instructions per DoF")
for o, n in c.most_common(40):
    print(f"{o:14s} {n / tot * 100:5.1f}%  {n * 32 / ndof:6.1f}/DoF")
