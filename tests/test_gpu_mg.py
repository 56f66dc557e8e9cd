"""GPU parity of the geometric multigrid against oracle/mg.py:
transfer operators, level eigenvalue estimates, one V-cycle, and MG-PCG
iteration counts (margin-guarded as R15)."""
import numpy as np
import pytest

import oracle
from oracle import mg
from tests._helpers import rel_l2, seeded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


CASES = [
    dict(n_cells=(4, 4, 4), k=2),
    dict(n_cells=(8, 4, 4), k=1, dirichlet=0b110011),
    dict(n_cells=(4, 6, 2), k=3, upper=(1.0, 1.5, 0.5)),
    dict(n_cells=(4, 4, 4), k=2, dirichlet=0b000001),  # one Dirichlet face
    dict(n_cells=(4, 4, 4), k=2, geometry="sine", coeff="variable"),
    dict(n_cells=(2, 2, 2), k=5),
]


def _kw(c):
    return dict(upper=c.get("upper", (1.0, 1.0, 1.0)), geom=1 if c.get("geometry") == "sine" else 0,
                coeff_kind=1 if c.get("coeff") == "variable" else 0, dirichlet=c.get("dirichlet"))


def _pair(c, torch, n_levels=0, max_coarse_dofs=60):
    from paper_1910_13247_b200 import Multigrid

    M = Multigrid(c["n_cells"], c["k"], upper=c.get("upper"), geometry=c.get("geometry", "cartesian"),
                  coeff=c.get("coeff", 1.0), dirichlet_faces=c.get("dirichlet"), n_levels=n_levels,
                  max_coarse_dofs=max_coarse_dofs)
    H = mg.build_hierarchy(3, c["n_cells"], c["k"], n_levels=M.n_levels, **_kw(c))
    assert [L.A.n for L in H.levels] == M.sizes
    return M, H


def _id(c):
    return f"k{c['k']}-{'x'.join(map(str, c['n_cells']))}-{c.get('geometry', 'cart')}-d{c.get('dirichlet')}"


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_transfer_and_lambda_match_oracle(case, torch):
    M, H = _pair(case, torch)
    for l in range(1, M.n_levels):
        xc = seeded(M.sizes[l - 1], 1)
        xf = seeded(M.sizes[l], 2)
        pf = M.prolongate(l, torch.from_numpy(xc).cuda()).cpu().numpy()
        assert np.abs(pf - mg.prolongate(H, l, xc)).max() <= 1e-14 * max(1.0, np.abs(xc).max())
        rc = M.restrict(l, torch.from_numpy(xf).cuda()).cpu().numpy()
        assert np.abs(rc - mg.restrict(H, l, xf)).max() <= 1e-13 * np.abs(xf).max()
        assert abs(M.level_lambda(l) - H.levels[l].lam) <= 1e-9 * H.levels[l].lam


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_vcycle_matches_oracle(case, torch):
    M, H = _pair(case, torch)
    mask = H.levels[-1].mask
    for s in (3, 4):
        b = seeded(M.n_local, s)
        b[mask] = 0.0
        v = M.vcycle(torch.from_numpy(b).cuda()).cpu().numpy()
        assert rel_l2(v, mg.vcycle(H, b)) <= 1e-12


def _margin_ok(hist, tol, normb):
    if len(hist) < 2:
        return True
    return min(hist[-2] / (tol * normb) - 1.0, 1.0 - hist[-1] / (tol * normb)) > 1e-6


@pytest.mark.parametrize("case", [CASES[0], CASES[2], CASES[4], dict(n_cells=(8, 8, 8), k=2)], ids=_id)
def test_mg_pcg_matches_oracle(case, torch):
    M, H = _pair(case, torch)
    b = oracle.rhs(H.levels[-1].p, 0)
    ref = mg.mg_pcg(H, b, 1e-10)
    x, res = M.cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-10)
    normb = np.linalg.norm(b)
    if _margin_ok(ref.history, 1e-10, normb):
        assert res.iterations == ref.iterations
    np.testing.assert_allclose(res.history, ref.history[:res.iterations], rtol=1e-6, atol=1e-13 * normb)
    assert rel_l2(x.cpu().numpy(), ref.x) <= 1e-8
    assert res.iterations <= 8


def test_mg_errors(torch):
    from paper_1910_13247_b200 import MFError, Multigrid

    with pytest.raises(MFError) as e:
        Multigrid((6, 4, 4), 2, n_levels=3)  # 6 not divisible by 4
    assert e.value.name == "MF_ERR_ARGUMENT"
    with pytest.raises(MFError) as e:
        Multigrid((16, 16, 16), 4, n_levels=1)  # coarse level above 2048 DoFs
    assert e.value.name == "MF_ERR_ARGUMENT"
    with pytest.raises(MFError) as e:
        Multigrid((4, 4, 4), 2, dirichlet_faces=0)  # pure Neumann: singular coarse operator
    assert e.value.name == "MF_ERR_SINGULAR"
    M = Multigrid((4, 4, 4), 2, n_levels=2)
    with pytest.raises(TypeError):
        M.vcycle(M.new_vector(0))


F32_CASES = [
    dict(dim=3, n_cells=(9, 10, 11), k=2),
    dict(dim=3, n_cells=(9, 17, 7), k=4, dirichlet=0b011001),
    dict(dim=3, n_cells=(9, 9, 13), k=3, upper=(1.0, 2.0, 0.5), coeff=3.0),
    dict(dim=3, n_cells=(5, 4, 6), k=3, geometry="sine", coeff="variable"),
    dict(dim=3, n_cells=(3, 3, 2), k=5),
    dict(dim=3, n_cells=(4, 3, 5), k=2, coeff="variable"),
]


@pytest.mark.parametrize("case", F32_CASES, ids=lambda c: f"k{c['k']}-{'x'.join(map(str, c['n_cells']))}")
def test_apply_f32_matches_oracle_to_single_precision(case, torch):
    # FP32 instance of the apply kernels (§8(f) f2): relative L2 error ~ (number of
    # rounded FP32 operations per output) x 2^-24; bound 2e-6 (x, A fixed in FP64)
    from tests._helpers import cuda_operator, oracle_problem

    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    x = seeded(A.n, 1).astype(np.float32)
    y = op.apply_f32(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    assert rel_l2(y, A @ x.astype(np.float64)) <= 2e-6


@pytest.mark.parametrize("case", [CASES[0], CASES[4], dict(n_cells=(8, 8, 8), k=2), dict(n_cells=(4, 4, 4), k=4)],
                         ids=_id)
def test_mixed_precision_mg_pcg(case, torch):
    # FP32 V-cycle inside the FP64 CG: the FP64 residual still reaches
    # 1e-10, within a couple of iterations of the FP64 V-cycle, same solution
    from paper_1910_13247_b200 import Multigrid

    M64, H = _pair(case, torch)
    M32 = Multigrid(case["n_cells"], case["k"], upper=case.get("upper"), geometry=case.get("geometry", "cartesian"),
                    coeff=case.get("coeff", 1.0), dirichlet_faces=case.get("dirichlet"), n_levels=M64.n_levels,
                    precision="mixed")
    b = oracle.rhs(H.levels[-1].p, 0)
    ref = mg.mg_pcg(H, b, 1e-10)
    x, res = M32.cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-10)
    assert res.final_rel_residual <= 1e-10
    assert res.iterations <= ref.iterations + 2
    assert rel_l2(x.cpu().numpy(), ref.x) <= 1e-8
