"""Time one operator's apply with CUDA events (kernel tuning; not a bench line).
python tools/time_apply.py --cells 64 --degree 5 [--geometry cartesian] [--coeff 1.0] [--reps 50]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", type=int, default=64)
ap.add_argument("--shape", default=None, help="nx,ny,nz (overrides --cells)")
ap.add_argument("--degree", type=int, default=5)
ap.add_argument("--geometry", default="cartesian")
ap.add_argument("--coeff", default="1.0")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--variant", default="auto")
ap.add_argument("--dirichlet", type=int, default=None)
a = ap.parse_args()
coeff = a.coeff if a.coeff == "variable" else float(a.coeff)
shape = tuple(int(v) for v in a.shape.split(",")) if a.shape else (a.cells,) * 3
op = Operator(shape, a.degree, geometry=a.geometry, coeff=coeff, dirichlet_faces=a.dirichlet)
if a.variant != "auto":
    op.set_variant(a.variant)
x = torch.from_numpy(synth.vector(op.n_local, 0)).cuda()
y = torch.empty_like(x)
for _ in range(5):
    op.apply(x, y)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(a.reps):
    op.apply(x, y)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.reps
print(f"k={a.degree} cells={shape} {a.geometry} c={a.coeff}: {ms * 1e3:.1f} us/apply, "
      f"{op.n_global / ms / 1e6:.2f} GDoF/s, variant {op.info()['apply_variant']}")
