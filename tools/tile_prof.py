"""Per-phase cycle breakdown of the tile kernel: MF_TILE_PROF=1 python tools/tile_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MF_TILE_PROF", "1")
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

op = Operator((64, 64, 64), 4)
x = torch.from_numpy(synth.vector(op.n_local, 0)).cuda()
y = torch.empty_like(x)
for _ in range(40):
    op.apply(x, y)
torch.cuda.synchronize()
