"""ncu driver: a few DG-SIP applies on the dg4 workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

op = Operator((64, 64, 64), 4, discretization="dg")
x = torch.from_numpy(synth.vector(op.n_local, 0)).cuda()
y = torch.empty_like(x)
for _ in range(4):
    op.apply(x, y)
torch.cuda.synchronize()
print("ok")
