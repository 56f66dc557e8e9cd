"""GPU parity of the solver path (§8(a) a10): eigenvalue estimate,
Chebyshev(6) preconditioner and Chebyshev-Jacobi PCG against the oracle's
numpy algorithms (O9-O11) driven by the oracle CSR SpMV.  CG iteration counts
must match exactly under the margin guard of R15."""
import numpy as np
import pytest

import oracle
import synth
from oracle import solvers
from tests._helpers import cuda_operator, oracle_problem, rel_l2, seeded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def _oracle_setup(case):
    p = oracle_problem(case)
    A = oracle.CSR(p)
    d = A.diagonal()
    s = synth.with_zero_dirichlet(synth.vector(A.n, 0), oracle.constrained_mask_fast(p))
    return p, A, d, s


CASES = [
    dict(dim=3, n_cells=(6, 5, 4), k=2),
    dict(dim=3, n_cells=(4, 4, 4), k=4),
    dict(dim=3, n_cells=(5, 4, 4), k=3, geometry="sine", coeff="variable"),
    dict(dim=2, n_cells=(4, 4), k=1),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['dim']}d-k{c['k']}-{c.get('geometry', 'cart')}")
def test_lambda_max_matches_oracle(case, torch):
    p, A, d, s = _oracle_setup(case)
    lam_ref = solvers.ritz_lambda_max(A.matvec, d, s, 12)
    lam = cuda_operator(case).estimate_lambda_max(12)
    assert abs(lam - lam_ref) <= 1e-9 * lam_ref


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['dim']}d-k{c['k']}-{c.get('geometry', 'cart')}")
@pytest.mark.parametrize("degree", [1, 2, 6])
def test_chebyshev_matches_oracle(case, degree, torch):
    p, A, d, s = _oracle_setup(case)
    op = cuda_operator(case)
    r = synth.with_zero_dirichlet(seeded(A.n, 3), oracle.constrained_mask_fast(p))
    lam = 1.2 * 1.7
    z_ref = solvers.chebyshev(A.matvec, d, r, lam, degree, 20.0)
    z = op.chebyshev(torch.from_numpy(r).cuda(), lam, degree, 20.0).cpu().numpy()
    assert rel_l2(z, z_ref) <= 1e-12


# more Chebyshev cases: anisotropic cells, Neumann and mixed faces, high degree (the k = 6 apply
# runs on the DMMA kernel)
MORE_CHEB_CASES = [
    dict(dim=3, n_cells=(5, 3, 4), k=3, dirichlet=0b100110, upper=(1.0, 2.0, 0.5), coeff=3.0),
    dict(dim=3, n_cells=(3, 2, 3), k=6, dirichlet=0b011001),
    dict(dim=3, n_cells=(4, 3, 2), k=4, dirichlet=0, lower=(-0.5, 0.0, 0.2), upper=(1.0, 0.7, 1.0)),
]


@pytest.mark.parametrize("case", MORE_CHEB_CASES, ids=lambda c: f"k{c['k']}-d{c['dirichlet']}")
@pytest.mark.parametrize("degree", [1, 6])
def test_chebyshev_more_cases(case, degree, torch):
    p, A, d, s = _oracle_setup(case)
    op = cuda_operator(case)
    r = synth.with_zero_dirichlet(seeded(A.n, 5), oracle.constrained_mask_fast(p))
    lam = 1.2 * op.estimate_lambda_max(12)
    z_ref = solvers.chebyshev(A.matvec, d, r, lam, degree, 20.0)
    z = op.chebyshev(torch.from_numpy(r).cuda(), lam, degree, 20.0).cpu().numpy()
    assert rel_l2(z, z_ref) <= 1e-12


def _margin_ok(hist, tol, normb):
    if len(hist) < 2:
        return True
    a = hist[-2] / (tol * normb) - 1.0
    b = 1.0 - hist[-1] / (tol * normb)
    return min(a, b) > 1e-6


SOLVE_CASES = [
    (dict(dim=3, n_cells=(16, 16, 16), k=2), "f1"),       # cfg 2, f = 1
    (dict(dim=3, n_cells=(16, 16, 16), k=2), "manufactured"),
    (dict(dim=3, n_cells=(16, 16, 16), k=2), "random"),
    (dict(dim=3, n_cells=(8, 8, 8), k=4), "random"),
    (dict(dim=3, n_cells=(8, 8, 8), k=3, geometry="sine", coeff="variable"), "f1"),  # cfg 4 shape, small
    (dict(dim=3, n_cells=(6, 6, 6), k=6), "f1"),
    (dict(dim=2, n_cells=(4, 4), k=1), "f1"),
]


@pytest.mark.parametrize("case,rhs", SOLVE_CASES, ids=lambda v: str(v) if isinstance(v, str) else f"k{v['k']}")
@pytest.mark.parametrize("tol", [1e-10, 1e-12])
def test_cg_iteration_counts_match_oracle(case, rhs, tol, torch):
    p, A, d, s = _oracle_setup(case)
    if rhs == "f1":
        b = oracle.rhs(p, 0)
    elif rhs == "manufactured":
        b = oracle.rhs(p, 1)
    else:
        b = synth.with_zero_dirichlet(seeded(A.n, 11), oracle.constrained_mask_fast(p))
    ref = solvers.chebyshev_pcg(A.matvec, d, b, s, rel_tol=tol)
    op = cuda_operator(case)
    x, res = op.cg_solve(torch.from_numpy(b).cuda(), rel_tol=tol)
    x = x.cpu().numpy()
    assert abs(res.lambda_max - ref.lambda_max) <= 1e-9 * ref.lambda_max
    normb = np.linalg.norm(b)
    if _margin_ok(ref.history, tol, normb):
        assert res.iterations == ref.iterations
    else:
        n = min(len(ref.history), res.iterations)
        np.testing.assert_allclose(res.history[:n], ref.history[:n], rtol=1e-8)
    # histories agree to 1e-6 relative above the round-off floor of the recursive
    # residual (|r| is only known to ~eps * cond(A) |b|; 1e-13 |b| covers cond <= 1e3)
    np.testing.assert_allclose(res.history, ref.history[:res.iterations], rtol=1e-6, atol=1e-13 * normb)
    assert rel_l2(x, ref.x) <= 1e-8
    assert res.final_rel_residual <= tol


def test_jacobi_pcg_matches_oracle(torch):
    case = dict(dim=3, n_cells=(8, 8, 8), k=2)
    p, A, d, s = _oracle_setup(case)
    b = oracle.rhs(p, 0)
    ref = solvers.pcg(A.matvec, b, lambda r: r / d, 1e-10)
    x, res = cuda_operator(case).cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-10, cheb_degree=0)
    assert res.iterations == ref.iterations
    assert rel_l2(x.cpu().numpy(), ref.x) < 1e-8


def test_manufactured_convergence_on_gpu(torch):
    # O(h^{k+1}) L2 convergence of the GPU solve (error measured by the oracle, Gauss k+3)
    errs = []
    for n in (4, 8):
        case = dict(dim=3, n_cells=(n, n, n), k=2)
        p = oracle_problem(case)
        b = oracle.rhs(p, 1)
        x, res = cuda_operator(case).cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-12)
        errs.append(oracle.l2_error(p, x.cpu().numpy()))
    assert abs(np.log2(errs[0] / errs[1]) - 3.0) < 0.1


def test_cg_errors(torch):
    from paper_1910_13247_b200 import MFError

    case = dict(dim=3, n_cells=(8, 8, 8), k=2)
    p = oracle_problem(case)
    b = torch.from_numpy(oracle.rhs(p, 0)).cuda()
    with pytest.raises(MFError) as e:
        cuda_operator(case).cg_solve(b, rel_tol=1e-14, max_iter=3)
    assert e.value.name == "MF_ERR_MAX_ITERATIONS"
    x, res = cuda_operator(case).cg_solve(torch.zeros_like(b))
    assert res.iterations == 0 and x.abs().max().item() == 0.0


@pytest.mark.parametrize("case", [dict(dim=3, n_cells=(16, 16, 16), k=2), dict(dim=3, n_cells=(8, 8, 8), k=4),
                                  dict(dim=3, n_cells=(8, 8, 8), k=3, geometry="sine", coeff="variable")],
                         ids=lambda c: f"k{c['k']}-{c.get('geometry', 'cart')}")
def test_mixed_precision_chebyshev_pcg(case, torch):
    # §8(f) f2 on the a10 path: the Chebyshev(6) preconditioner in FP32 inside the FP64 CG
    # (the preconditioner changes by O(1e-7), CG keeps the FP64 residual recursion): the
    # FP64 stopping test is met, in at most two more iterations than the FP64 oracle run
    p, A, d, s = _oracle_setup(case)
    b = oracle.rhs(p, 0)
    ref = solvers.chebyshev_pcg(A.matvec, d, b, s, rel_tol=1e-10)
    op = cuda_operator(case)
    x, res = op.cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-10, precision="mixed")
    assert res.final_rel_residual <= 1e-10
    assert ref.iterations - 1 <= res.iterations <= ref.iterations + 2, (res.iterations, ref.iterations)
    assert rel_l2(x.cpu().numpy(), ref.x) <= 1e-8
    assert abs(res.lambda_max - ref.lambda_max) <= 1e-9 * ref.lambda_max
