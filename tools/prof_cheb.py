"""ncu driver: one Chebyshev(6) preconditioner application on cfg3 (fused steps unless MF_CHEB_FUSED=0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

nc, k, geom, coeff, _ = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
op = Operator(nc, k, geometry=geom, coeff=coeff)
r = torch.from_numpy(synth.vector(op.n_local, 3)).cuda()
for _ in range(2):
    z = op.chebyshev(r, 2.0, 6, 20.0)
torch.cuda.synchronize()
print("ok", float(z.norm()))
