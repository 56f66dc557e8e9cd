"""Worker of tests/test_gpu_multi.py (run under torchrun, one rank per GPU, NCCL): every rank
builds its z-slab Operator over the process group, applies it to its slice of one seeded global
vector, forms the diagonal and runs the Chebyshev-PCG; rank 0 gathers the slices and compares
them with the assembled oracle (both copies of a shared plane must agree bitwise).  Prints one
JSON line on rank 0."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from oracle import solvers  # noqa: E402
from tests._helpers import cuda_operator, oracle_problem, rel_l2, seeded  # noqa: E402
import synth  # noqa: E402

case = json.loads(sys.argv[1])
case["n_cells"] = tuple(case["n_cells"])
rank = int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl")
op = cuda_operator(case, group=dist.group.WORLD)
p = oracle_problem(case)
N = op.n_global
x = seeded(N, 1)
sl = slice(op.first_global, op.first_global + op.n_local)
y = op.apply(torch.from_numpy(x[sl].copy()).cuda()).cpu().numpy()
d = op.diagonal().cpu().numpy()
mask = oracle.constrained_mask_fast(p)
b = synth.with_zero_dirichlet(synth.vector(N, 4), mask)
_, res = op.cg_solve(torch.from_numpy(b[sl].copy()).cuda(), rel_tol=1e-10)
parts = [None] * dist.get_world_size()
dist.all_gather_object(parts, (op.first_global, y, d, res.iterations))
if rank == 0:
    A = oracle.CSR(p)
    y_ref, d_ref = A @ x, A.diagonal()
    # the Ritz start vector of mf_estimate_lambda_max (tests/test_gpu_solver.py::_oracle_setup)
    s = synth.with_zero_dirichlet(synth.vector(N, 0), mask)
    ref = solvers.chebyshev_pcg(A.matvec, d_ref, b, s, rel_tol=1e-10)
    from tests.test_gpu_solver import _margin_ok

    out = {"apply_err": 0.0, "diag_err": 0.0, "shared_planes_equal": True, "iterations": [], "oracle_iterations":
           ref.iterations, "margin_ok": bool(_margin_ok(ref.history, 1e-10, np.linalg.norm(b)))}
    gy, gd = np.zeros(N), np.zeros(N)
    for i, (fg, yy, dd, it) in enumerate(parts):
        out["apply_err"] = max(out["apply_err"], rel_l2(yy, y_ref[fg:fg + len(yy)]))
        out["diag_err"] = max(out["diag_err"], rel_l2(dd, d_ref[fg:fg + len(dd)]))
        out["iterations"].append(it)
        if i > 0:  # the shared plane: this rank's first = the previous rank's last
            pf, py, _, _ = parts[i - 1]
            n_sh = pf + len(py) - fg
            out["shared_planes_equal"] &= bool(np.array_equal(yy[:n_sh], py[-n_sh:]))
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
