"""Small driver for ncu captures: build one operator and run a few applies.
python tools/prof_apply.py [--config cfg3] [--variant auto] [--reps 5] [--cells n]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--variant", default="auto")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cells", type=int, default=0, help="override: n^3 cells")
a = ap.parse_args()
nc, k, geom, coeff, _ = CONFIGS[a.config]
if a.cells:
    nc = (a.cells,) * 3
if geom == "hex":
    from bench import make_hex_operator

    op, _ = make_hex_operator(nc, k, coeff, torch.cuda.current_device())
elif geom == "dg":
    op = Operator(nc, k, coeff=coeff, discretization="dg")
else:
    op = Operator(nc, k, geometry=geom, coeff=coeff)
    op.set_variant(a.variant)
x = torch.from_numpy(synth.vector(op.n_local, 0)).cuda()
y = torch.empty_like(x)
for _ in range(a.reps):
    op.apply(x, y)
torch.cuda.synchronize()
print("ok", op.info())
