"""Per-SASS-instruction stall samples (top N) of an ncu report:
python tools/ncu_sassstall.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si, ss, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [(i, k) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[ss] or 0), int(r[ei] or 0), r[0][-5:], r[si].strip(), r))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for smp, n, a, src, r in sorted(data, key=lambda d: -d[0])[:top]:
    rs = sorted(((int(r[i] or 0), k[6:]) for i, k in reasons), reverse=True)[:2]
    print(f"{smp / tot * 100:5.2f}% {a} n={n:9d} {src[:60]:60s} " + " ".join(f"{k}={v * 100 / tot:.2f}" for v, k in rs))
