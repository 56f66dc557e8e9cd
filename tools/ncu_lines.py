"""Per-phase / per-line stall and instruction shares of an ncu source export (cuda,sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
srcf = sys.argv[2]
res = []
tot_s = tot_i = 0
for r in rows[3:]:
    if r and r[0].strip().isdigit() and len(r) > 7:
        try:
            s, i = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        res.append((int(r[0]), r[1][:90], s, i))
        tot_s += s
        tot_i += i
src = open(srcf).read().split('\n')
keys = [('---- phase A', 'A'), ('---- phase B', 'B'), ('---- phase C', 'C'), ('auto prefetch', 'prefetch'),
        ('auto columns_of', 'columns'), ('auto item_of', 'item'), ('void eo_split', 'eo_split'),
        ('void eo_acc', 'eo_acc'), ('void eo_first', 'eo_first'), ('void eo_combine', 'eo_combine'),
        ('void cp_async8', 'cp_async'), ('while (true)', 'item-setup')]


def phase(ln):
    for k in range(ln - 1, -1, -1):
        for key, name in keys:
            if key in src[k]:
                return name
    return 'other'


agg = {}
for ln, txt, s, i in res:
    a = agg.setdefault(phase(ln), [0, 0])
    a[0] += s
    a[1] += i
for p, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{p:12s} stall {100 * s / tot_s:5.1f}%  instr {100 * i / tot_i:5.1f}%")
res.sort(key=lambda x: -x[2])
for ln, txt, s, i in res[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    print(f"{ln:4d} {100 * s / tot_s:5.1f}% {100 * i / tot_i:5.1f}% {txt}")
