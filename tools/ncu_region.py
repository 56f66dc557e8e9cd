"""Stall samples of an ncu report split by source-line region (producer / consumer of the halo
kernel) with per-reason shares and the top lines of each region:
python tools/ncu_region.py report.ncu-rep csrc_file [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, srcf = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
src = open(srcf).read().split("\n")
pl = next(i + 1 for i, l in enumerate(src) if "producer warps: y step" in l)
cl = next(i + 1 for i, l in enumerate(src) if "consumer warps: x and z steps" in l)
el = next(i + 1 for i, l in enumerate(src) if "no CTA leaves while" in l)
fname = srcf.split("/")[-1]
h = None
cur = None
agg = collections.defaultdict(collections.Counter)
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or not r or not r[0]:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (cur, ln)
    for k, i in h.items():
        if k.startswith("stall_") or k in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                agg[key][k] += int(r[i] or 0)
            except (ValueError, IndexError):
                pass
S = "Warp Stall Sampling (All Samples)"
tot = sum(c[S] for c in agg.values()) or 1


def region(key):
    f, ln = key
    if f != fname:
        return "inlined helpers"
    return "producer" if pl <= ln < cl else ("consumer" if cl <= ln < el else "other")


reg = collections.defaultdict(collections.Counter)
for k, c in agg.items():
    reg[region(k)].update(c)
for name, c in reg.items():
    reasons = sorted(((v, k) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:6]
    print(f"{name:16s} samples {c[S] / tot * 100:5.1f}%  inst {c['Instructions Executed']}  " +
          " ".join(f"{k[6:]}={v / tot * 100:.1f}" for v, k in reasons))
for name in ("other", "consumer", "producer"):
    print("== top lines:", name)
    lines = sorted(((c[S], k) for k, c in agg.items() if region(k) == name), reverse=True)[:top]
    for v, (f, ln) in lines:
        c = agg[(f, ln)]
        reasons = sorted(((x, k) for k, x in c.items() if k.startswith("stall_")), reverse=True)[:3]
        print(f"  {v / tot * 100:5.1f} {ln:4d} {src[ln - 1].strip()[:70]:70s} " +
              " ".join(f"{k[6:]}={x / tot * 100:.1f}" for x, k in reasons))
