"""Per-source-line stall / instruction shares from `ncu -i X --page source --csv --print-source cuda,sass`.
python tools/ncu_srcstall.py export.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = "?"
h = None
agg = {}
reasons = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_long_sb", "stall_math", "stall_mio",
           "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_wait", "stall_lg"]
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        if h is None:
            h = {}
            for i, k in enumerate(r):
                h.setdefault(k, i)
        continue
    if h is None or len(r) < 40 or not r[0]:
        continue
    try:
        key = (f, int(r[0]), r[1][:70])
        int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(key, [0, 0] + [0] * len(reasons))
    a[0] += int(r[4] or 0)
    a[1] += int(r[7] or 0)
    for j, rs in enumerate(reasons):
        a[2 + j] += int(r[h[rs]] or 0)
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"total samples {ts}, warp instr {ti}")
print("stall%  inst%  " + " ".join(x.replace("stall_", "")[:6] for x in reasons))
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{a[0]/ts*100:5.1f} {a[1]/ti*100:5.1f}  " + " ".join(f"{x/ts*100:6.1f}" for x in a[2:]) + f"  {k[0][:12]}:{k[1]} {k[2]}")
