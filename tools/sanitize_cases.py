"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck; one tool per run):  compute-sanitizer --tool T python tools/sanitize_cases.py
halo (k=4, 1-3 CTA clusters, z chunks with halo, split parts, host pipeline), plane (k=2,3),
cell3 (Cartesian Q6 padded, curved Q3 with TMA metric staging), general 2D, hex (constraint
lines), DG (k=4), multigrid transfers + V-cycle + MG-PCG, FP32 apply, fused CG."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1910_13247_b200 import Multigrid, Operator  # noqa: E402


def run(op, label):
    x = torch.from_numpy(synth.vector(op.n_local, 1)).cuda()
    y = op.apply(x)
    torch.cuda.synchronize()
    print(f"{label}: |Ax| = {y.norm().item():.6e}", flush=True)
    return op


for nc, d in (((9, 17, 7), None), ((40, 7, 5), 0), ((70, 3, 5), 0b100110)):
    run(Operator(nc, 4, dirichlet_faces=d), f"halo {nc}")
op = Operator((40, 7, 5), 4, dirichlet_faces=0)
x = torch.from_numpy(synth.vector(op.n_local, 2)).cuda()
y = op.new_vector()
op.apply_split_part(x, y, 1)
op.apply_split_part(x, y, 2)
torch.cuda.synchronize()
print("halo split parts ok", flush=True)
os.environ["MF_HOST_PIPELINE"] = "3"
op = Operator((9, 5, 12), 4)
op.apply_host(synth.vector(op.n_local, 3))
print("halo host pipeline ok", flush=True)
del os.environ["MF_HOST_PIPELINE"]
for k in (2, 3):
    op = Operator((9, 10, 7), k)
    op.set_variant("plane")
    run(op, f"plane k={k}")
run(Operator((4, 3, 5), 6), "cell3 cartesian Q6")
run(Operator((6, 5, 4), 3, geometry="sine", coeff="variable"), "cell3 curved Q3")
run(Operator((7, 5), 3, dim=2), "general 2D Q3")
run(Operator((5, 4, 3), 4, discretization="dg"), "DG Q4")
# unstructured hex with a 2:1 interface (constraint lines)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import _hexmesh as hm  # noqa: E402
from paper_1910_13247_b200 import HexOperator  # noqa: E402

m = hm.two_block((2, 2, 1), 2, 3)
run(HexOperator(m["vertices"], m["cells"], m["k"], m["cell_dofs"], m["n_dofs"], m["lines"], m["dirichlet"]),
    "hex Q3 with hanging lines")
M = Multigrid((8, 8, 8), 2)
b = torch.ones(M.sizes[-1], dtype=torch.float64, device="cuda")
xs, res = M.cg_solve(b, rel_tol=1e-8)
print(f"MG-PCG: {res.iterations} iterations", flush=True)
M.close()
op = Operator((6, 6, 6), 2)
xs, res = op.cg_solve(torch.ones(op.n_local, dtype=torch.float64, device="cuda"), rel_tol=1e-8)
print(f"Chebyshev-PCG: {res.iterations} iterations", flush=True)
xf = op.apply_f32(torch.ones(op.n_local, dtype=torch.float32, device="cuda"))
torch.cuda.synchronize()
print("sanitize cases done", flush=True)
