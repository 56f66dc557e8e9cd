"""GPU parity of the z-slab decomposition (§8(a) a8 / §8(e); §3.1, the
distributed mesh) on one GPU, with detached slab operators (mf_dist with world_size > 1 and no
NCCL unique id): every rank's operator is built exactly as in a distributed run (partition,
interior z faces unconstrained, identity rows of a shared plane written by the upper rank) and
applied to its slice of one global vector on the GPU; the test then performs the exchange the
library does over NCCL (each rank adds its neighbour's partial sums on the shared planes,
api.cu::halo_post / halo_add) and compares every rank's result with the assembled oracle.
The ranks run one after another -- no kernel waits on another rank -- so only the transport
(ncclSend / ncclRecv of a contiguous plane) is left to the multi-GPU run."""
import numpy as np
import pytest

import oracle
from tests._helpers import CUDA_ORACLE_TOL, cuda_operator, oracle_problem, rel_l2, seeded

pytestmark = pytest.mark.gpu

CASES = [
    (dict(dim=3, n_cells=(5, 4, 8), k=4), 2),                                  # halo kernel
    (dict(dim=3, n_cells=(5, 4, 8), k=4), 4),
    (dict(dim=3, n_cells=(40, 7, 9), k=4, dirichlet=0), 3),                    # 2-CTA cluster, Neumann
    (dict(dim=3, n_cells=(6, 5, 7), k=2, dirichlet=0b011001), 3),              # plane kernel
    (dict(dim=3, n_cells=(3, 2, 6), k=6), 2),                                  # DMMA kernel
    (dict(dim=3, n_cells=(3, 2, 6), k=6, dirichlet=0b110011, upper=(1.0, 2.0, 0.5)), 3),
    (dict(dim=3, n_cells=(4, 3, 6), k=3, geometry="sine", coeff="variable"), 2),  # curved, stored metric
    (dict(dim=3, n_cells=(4, 4, 5), k=1, dirichlet=0b100000), 5),              # one layer per rank
]


def _id(v):
    case, world = v if isinstance(v, tuple) else (v, None)
    return f"k{case['k']}-{'x'.join(map(str, case['n_cells']))}-d{case.get('dirichlet')}-P{world}"


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.parametrize("cw", CASES, ids=_id)
def test_slab_decomposition_matches_oracle(cw, torch):
    case, world = cw
    p = oracle_problem(case)
    A = oracle.CSR(p)
    mask = oracle.constrained_mask_fast(p)
    ops = [cuda_operator(case, slab=(r, world)) for r in range(world)]
    plane = ops[0].n_local - ops[0].n_owned if world > 1 else 0
    assert all(op.n_global == A.n for op in ops)
    assert ops[-1].first_global + ops[-1].n_local == A.n
    for s in (1, 2):
        x = seeded(A.n, s)
        y_ref = A @ x
        part = []
        for op in ops:  # each rank's apply on its slice: partial sums on the shared planes
            xl = torch.from_numpy(x[op.first_global:op.first_global + op.n_local].copy()).cuda()
            part.append(op.apply(xl).cpu().numpy())
        for r, op in enumerate(ops):  # the exchange: add the neighbour's partial of each shared plane
            y = part[r].copy()
            if r > 0:
                y[:plane] += part[r - 1][-plane:]
            if r < world - 1:
                y[-plane:] += part[r + 1][:plane]
            sl = slice(op.first_global, op.first_global + op.n_local)
            assert rel_l2(y, y_ref[sl]) <= CUDA_ORACLE_TOL, (r, s, rel_l2(y, y_ref[sl]))
            np.testing.assert_array_equal(y[mask[sl]], x[sl][mask[sl]])


@pytest.mark.parametrize("cw", [CASES[0], CASES[3], CASES[5], CASES[6]], ids=_id)
def test_slab_diagonal_matches_oracle(cw, torch):
    # mf_diagonal of a detached slab: partial sums on the shared planes, exchanged by the test
    case, world = cw
    p = oracle_problem(case)
    d_ref = oracle.CSR(p).diagonal()
    ops = [cuda_operator(case, slab=(r, world)) for r in range(world)]
    plane = ops[0].n_local - ops[0].n_owned
    part = [op.diagonal().cpu().numpy() for op in ops]
    for r, op in enumerate(ops):
        d = part[r].copy()
        if r > 0:
            d[:plane] += part[r - 1][-plane:]
        if r < world - 1:
            d[-plane:] += part[r + 1][:plane]
        sl = slice(op.first_global, op.first_global + op.n_local)
        assert rel_l2(d, d_ref[sl]) <= CUDA_ORACLE_TOL


def test_slab_partition_matches_mf_partition(torch):
    from paper_1910_13247_b200.mf import partition

    case = dict(dim=3, n_cells=(3, 4, 10), k=3)
    for world in (2, 3, 5):
        for r in range(world):
            op = cuda_operator(case, slab=(r, world))
            part = partition(case["n_cells"], case["k"], r, world)
            assert (op.first_global, op.n_local, op.n_owned) == (part["first_global"], part["n_local"],
                                                                  part["n_owned"])


def test_slab_apply_host_equals_device_apply(torch):
    # mf_apply_host on a slab (the non-pipelined host path, as the bench's e2e leg at N > 1)
    case = dict(dim=3, n_cells=(5, 4, 8), k=4, dirichlet=0b011001)
    for r in range(3):
        op = cuda_operator(case, slab=(r, 3))
        x = seeded(op.n_global, 4)[op.first_global:op.first_global + op.n_local].copy()
        yd = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        np.testing.assert_array_equal(op.apply_host(x), yd)


def test_detached_slab_refuses_collectives(torch):
    from paper_1910_13247_b200 import MFError

    op = cuda_operator(dict(dim=3, n_cells=(3, 3, 4), k=2), slab=(0, 2))
    b = torch.ones(op.n_local, dtype=torch.float64, device="cuda")
    with pytest.raises(MFError):
        op.cg_solve(b)
    with pytest.raises(MFError):
        op.estimate_lambda_max(5)
    with pytest.raises(MFError):
        op.chebyshev(b, 2.0, 3, 20.0)
