"""GPU parity of the owner-writes Q4 kernel (apply variant 6, kernels_halo.cu) against the
assembled CPU oracle (§8(a) a3-a7, R11: relative L2 <= 1e-12; identity rows bitwise).

The kernel has no init pass and no atomics: every output node is stored once by the CTA
that owns it, the y halo of a tile and the z halo of a chunk are recomputed, and the x
halo crosses the thread-block cluster through distributed shared memory.  The cases cover
one to eight CTAs per cluster (n_cells x 1..256), full and partial last tiles in x and y,
many z-chunks (each chunk above layer 0 recomputes the layer below), anisotropic cells,
Neumann faces, the z-split launch order of the multi-GPU overlap (parts 1 + 2) and the
pipelined host apply (part 3, layer ranges)."""
import numpy as np
import pytest

import oracle
from tests._helpers import CUDA_ORACLE_TOL, cuda_operator, oracle_problem, rel_l2, seeded

pytestmark = pytest.mark.gpu

HALO_CASES = [
    dict(dim=3, n_cells=(1, 1, 1), k=4),
    dict(dim=3, n_cells=(9, 17, 7), k=4),                                   # one CTA, partial tiles
    dict(dim=3, n_cells=(5, 3, 20), k=4, dirichlet=0),                      # Neumann, many z-chunks
    dict(dim=3, n_cells=(4, 8, 5), k=4, dirichlet=0b011001),                # x+ Neumann (partial CTA)
    dict(dim=3, n_cells=(32, 4, 6), k=4),                                   # one full CTA: x+ column identity
    dict(dim=3, n_cells=(33, 5, 7), k=4),                                   # 32 + 1 cells: two CTAs
    dict(dim=3, n_cells=(40, 7, 11), k=4, dirichlet=0),                     # two CTAs, all Neumann
    dict(dim=3, n_cells=(64, 4, 9), k=4),                                   # two full CTAs (cfg 3 x extent)
    dict(dim=3, n_cells=(70, 3, 5), k=4, dirichlet=0b100110),               # three CTAs, mixed faces
    dict(dim=3, n_cells=(45, 6, 8), k=4, upper=(1.0, 2.0, 0.5), coeff=3.0),  # anisotropic cells
    dict(dim=3, n_cells=(20, 9, 13), k=4, lower=(-0.5, 0.0, 0.2), upper=(1.0, 0.7, 1.0), dirichlet=0b010111),
    dict(dim=3, n_cells=(256, 2, 3), k=4),                                  # eight CTAs: the largest cluster
    dict(dim=3, n_cells=(3, 2, 40), k=4, dirichlet=0b001111),               # z Neumann, long z
]


def _id(c):
    return f"{'x'.join(map(str, c['n_cells']))}-d{c.get('dirichlet')}-c{c.get('coeff', 1.0)}"


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _check(case, torch, seeds=(1, 2, 3), host=False):
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    op.set_variant("halo")
    assert op.info()["apply_variant"] == 6
    for s in seeds:
        x = seeded(A.n, s)
        y_ref = A @ x
        if host:
            y = op.apply_host(x)
        else:
            y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        err = rel_l2(y, y_ref)
        assert err <= CUDA_ORACLE_TOL, (s, err)
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])
    return op


@pytest.mark.parametrize("case", HALO_CASES, ids=_id)
def test_halo_kernel_matches_oracle(case, torch):
    _check(case, torch)


def test_halo_is_the_default_for_q4(torch):
    op = cuda_operator(dict(dim=3, n_cells=(8, 8, 8), k=4))
    assert op.info()["apply_variant"] == 6


@pytest.mark.parametrize("case", [HALO_CASES[2], HALO_CASES[6], HALO_CASES[8], HALO_CASES[12]], ids=_id)
def test_halo_zsplit_parts_match_oracle(case, torch, monkeypatch):
    # the multi-GPU overlap order (boundary layers, then the interior; §8(e)) on one GPU
    monkeypatch.setenv("MF_ZSPLIT", "1")
    _check(case, torch, seeds=(1, 2))


@pytest.mark.parametrize("case,chunks", [(HALO_CASES[2], "4"), (HALO_CASES[6], "3"), (HALO_CASES[12], "8")],
                         ids=lambda v: v if isinstance(v, str) else _id(v))
def test_halo_pipelined_host_apply(case, chunks, torch, monkeypatch):
    # mf_apply_host by z cell-layer ranges: each range's chunk above layer 0 reads the layer
    # below (uploaded with the previous range) and writes only its own planes
    monkeypatch.setenv("MF_HOST_PIPELINE", chunks)
    _check(case, torch, seeds=(1, 2), host=True)


def test_halo_unsupported_cases_are_rejected(torch):
    from paper_1910_13247_b200 import MFError

    for case in (dict(dim=3, n_cells=(32, 3, 3), k=4, dirichlet=0),    # full last CTA, x+ Neumann
                 dict(dim=3, n_cells=(5, 4, 3), k=4, dirichlet=0),     # full top tile, y+ Neumann
                 dict(dim=3, n_cells=(257, 2, 2), k=4),                # cluster of 9 CTAs
                 dict(dim=3, n_cells=(5, 5, 5), k=3)):
        op = cuda_operator(case)
        assert op.info()["apply_variant"] != 6
        with pytest.raises(MFError):
            op.set_variant("halo")


def test_halo_cfg3_full_size_vs_kronecker_oracle(torch):
    # BASELINE configs[2] (Q4 on 64^3, 16,974,593 DoFs) in the bench launch configuration
    case = dict(dim=3, n_cells=(64, 64, 64), k=4)
    p = oracle_problem(case)
    op = cuda_operator(case)
    assert op.info()["apply_variant"] == 6
    x = seeded(op.n_local, 1)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    y_ref = oracle.kron_apply(p, x)
    assert rel_l2(y, y_ref) <= CUDA_ORACLE_TOL
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


SPLIT_CASES = [
    (dict(dim=3, n_cells=(9, 17, 7), k=4), "halo"),
    (dict(dim=3, n_cells=(40, 7, 11), k=4, dirichlet=0), "halo"),
    (dict(dim=3, n_cells=(70, 3, 9), k=4, dirichlet=0b100110), "halo"),
    (dict(dim=3, n_cells=(9, 10, 11), k=2), "plane"),
    (dict(dim=3, n_cells=(6, 5, 7), k=3, geometry="sine", coeff="variable"), "general"),
    (dict(dim=3, n_cells=(3, 3, 5), k=5), "general"),
]


@pytest.mark.parametrize("case,variant", SPLIT_CASES, ids=lambda v: v if isinstance(v, str) else _id(v))
def test_split_interior_part_never_touches_the_shared_planes(case, variant, torch):
    # §8(e) overlap: part 2 (interior layers) runs while NCCL reads the partial sums of the
    # shared z-planes (the first and last plane of the local vector), so it must neither write
    # them nor need them; part 1 + part 2 = mf_apply.  A finite sentinel pattern catches plain
    # stores and atomic adds alike.
    op = cuda_operator(case)
    op.set_variant(variant)
    n = op.n_local
    plane = (case["k"] * case["n_cells"][0] + 1) * (case["k"] * case["n_cells"][1] + 1)
    x = torch.from_numpy(seeded(n, 3)).cuda()
    sentinel = torch.arange(n, dtype=torch.float64, device="cuda") * 1e-3 + 12345.0
    dst = sentinel.clone()
    op.apply_split_part(x, dst, 2)
    torch.cuda.synchronize()
    assert torch.equal(dst[:plane], sentinel[:plane])
    assert torch.equal(dst[-plane:], sentinel[-plane:])
    # part 2 did write the interior (it is not a no-op) when there are interior layers
    if case["n_cells"][2] > 2:
        assert not torch.equal(dst[plane:-plane], sentinel[plane:-plane])
    ref = op.apply(x)
    both = sentinel.clone()
    op.apply_split_part(x, both, 1)
    op.apply_split_part(x, both, 2)
    err = ((both - ref).norm() / ref.norm()).item()
    assert err <= (0.0 if variant == "halo" else 1e-14), err


def test_binding_argument_checks(torch):
    op = cuda_operator(dict(dim=3, n_cells=(2, 2, 2), k=2))
    x = seeded(op.n_local, 1)
    with pytest.raises(TypeError):
        op.apply_host(x, np.empty(op.n_local, dtype=np.float32))
    with pytest.raises(TypeError):
        op.apply_host(x, np.empty(2 * op.n_local)[::2])
    with pytest.raises(TypeError):
        op.apply(torch.from_numpy(x))  # a CPU tensor
    op.sync()
