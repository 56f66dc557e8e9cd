"""GPU parity of the FP64 tensor-core cell kernel (kernels_tc.cu::k_apply_tc: Cartesian,
constant coefficient, k = 5..7, the default for those operators) against the assembled CPU
oracle (§8(a) a3-a7, R11: relative L2 <= 1e-12; identity rows bitwise).

One warp walks a column of cells along z in chunks; consecutive cells of a chunk reuse the
shared z-face slice and carry its partial sums in registers, chunk boundaries meet by atomic
adds.  The cases cover single- and multi-chunk columns (n_z >= 8 splits into chunks of >= 4
cells), every Dirichlet / Neumann face mix, anisotropic cells, the z-split launch order of the
multi-GPU overlap (parts 1 + 2) and the pipelined host apply (cell-layer ranges)."""
import numpy as np
import pytest

import oracle
from tests._helpers import CUDA_ORACLE_TOL, cuda_operator, oracle_problem, rel_l2, seeded

pytestmark = pytest.mark.gpu

TC_CASES = [
    dict(dim=3, n_cells=(1, 1, 1), k=6),
    dict(dim=3, n_cells=(2, 3, 4), k=6),
    dict(dim=3, n_cells=(3, 2, 17), k=6),                                     # chunks of 5 + ragged
    dict(dim=3, n_cells=(2, 2, 24), k=6, dirichlet=0),                        # Neumann, 6 chunks
    dict(dim=3, n_cells=(3, 3, 12), k=6, dirichlet=0b011001),
    dict(dim=3, n_cells=(4, 2, 9), k=6, dirichlet=0b100110, upper=(1.0, 2.0, 0.5), coeff=3.0),
    dict(dim=3, n_cells=(2, 3, 10), k=6, lower=(-0.5, 0.0, 0.2), upper=(1.0, 0.7, 1.0), dirichlet=0b010111),
    dict(dim=3, n_cells=(3, 3, 2), k=5),
    dict(dim=3, n_cells=(2, 3, 16), k=5, dirichlet=0b001111),
    dict(dim=3, n_cells=(2, 2, 1), k=7),
    dict(dim=3, n_cells=(2, 2, 9), k=7, dirichlet=0b110000, upper=(0.5, 1.0, 1.5)),
]


def _id(c):
    return f"k{c['k']}-{'x'.join(map(str, c['n_cells']))}-d{c.get('dirichlet')}-c{c.get('coeff', 1.0)}"


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _check(case, torch, seeds=(1, 2, 3), host=False):
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    for s in seeds:
        x = seeded(A.n, s)
        y_ref = A @ x
        y = op.apply_host(x) if host else op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        err = rel_l2(y, y_ref)
        assert err <= CUDA_ORACLE_TOL, (s, err)
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


@pytest.mark.parametrize("case", TC_CASES, ids=_id)
def test_tc_kernel_matches_oracle(case, torch):
    _check(case, torch)


@pytest.mark.parametrize("case", [TC_CASES[2], TC_CASES[3], TC_CASES[8]], ids=_id)
def test_tc_zsplit_parts_match_oracle(case, torch, monkeypatch):
    monkeypatch.setenv("MF_ZSPLIT", "1")
    _check(case, torch, seeds=(1, 2))


@pytest.mark.parametrize("case,chunks", [(TC_CASES[2], "4"), (TC_CASES[3], "3")],
                         ids=lambda v: v if isinstance(v, str) else _id(v))
def test_tc_pipelined_host_apply(case, chunks, torch, monkeypatch):
    monkeypatch.setenv("MF_HOST_PIPELINE", chunks)
    _check(case, torch, seeds=(1, 2), host=True)


def test_tc_split_interior_part_never_touches_the_shared_planes(torch):
    case = dict(dim=3, n_cells=(2, 3, 11), k=6, dirichlet=0b100110)
    op = cuda_operator(case)
    n = op.n_local
    plane = (6 * 2 + 1) * (6 * 3 + 1)
    x = torch.from_numpy(seeded(n, 3)).cuda()
    sentinel = torch.arange(n, dtype=torch.float64, device="cuda") * 1e-3 + 12345.0
    dst = sentinel.clone()
    op.apply_split_part(x, dst, 2)
    torch.cuda.synchronize()
    assert torch.equal(dst[:plane], sentinel[:plane])
    assert torch.equal(dst[-plane:], sentinel[-plane:])
    ref = op.apply(x)
    both = sentinel.clone()
    op.apply_split_part(x, both, 1)
    op.apply_split_part(x, both, 2)
    assert ((both - ref).norm() / ref.norm()).item() <= 1e-14
