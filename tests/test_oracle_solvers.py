"""Pins for the oracle solvers (O9-O11) and the manufactured-solution
convergence of the oracle discretisation (O8): textbook CG properties, exact
Lanczos, the closed-form Chebyshev residual polynomial, and O(h^{k+1}) L2
convergence (north star)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import solvers


def test_cg_identity_one_iteration():
    b = synth.vector(50, 1)
    r = solvers.pcg(lambda x: x.copy(), b, lambda r: r.copy(), 1e-12)
    assert r.iterations == 1
    np.testing.assert_allclose(r.x, b, rtol=1e-15)


def test_cg_diag_finite_termination():
    d = np.arange(1.0, 11.0)
    b = np.ones(10)
    r = solvers.pcg(lambda x: d * x, b, lambda r: r.copy(), 1e-12)
    assert r.iterations <= 10
    np.testing.assert_allclose(r.x, b / d, rtol=1e-10)


def test_cg_breakdown_on_indefinite():
    d = np.array([1.0, -1.0, 2.0])
    with pytest.raises(solvers.BreakdownError):
        solvers.pcg(lambda x: d * x, np.array([0.0, 1.0, 0.0]), lambda r: r.copy(), 1e-12)


def test_cg_max_iterations():
    d = np.arange(1.0, 101.0)
    with pytest.raises(solvers.MaxIterationsError):
        solvers.pcg(lambda x: d * x, np.ones(100), lambda r: r.copy(), 1e-14, max_iter=3)


def test_pcg_jacobi_matches_dense_solve_q1_16x16():
    # assembled Q1 Laplace on 16x16 with Jacobi -> dense factorisation to 1e-8
    p = oracle.problem(dim=2, n_cells=(16, 16), degree=1)
    A = oracle.CSR(p)
    b = oracle.rhs(p, 0)
    d = A.diagonal()
    r = solvers.pcg(A.matvec, b, lambda r: r / d, 1e-12)
    np.testing.assert_allclose(r.x, np.linalg.solve(A.dense(), b), rtol=0, atol=1e-8 * np.abs(r.x).max())


def test_ritz_exact_for_few_distinct_eigenvalues():
    # diag(1..10): 12 CG-Lanczos steps recover lambda_max = 10 exactly (estimate in [9.5,12] after x1.2)
    d = np.arange(1.0, 11.0)
    s = synth.vector(10, 0)
    lam = solvers.ritz_lambda_max(lambda x: d * x, np.ones(10), s, 12)
    assert abs(lam - 10.0) < 1e-10
    assert 9.5 <= 1.2 * lam <= 12.0


def test_ritz_equals_explicit_lanczos():
    # independent: explicit Lanczos with full re-orthogonalisation on D^{-1/2} A D^{-1/2}
    rng = np.random.default_rng(5)
    n = 60
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = Q @ np.diag(np.linspace(0.5, 40, n)) @ Q.T
    dg = np.diag(A).copy()
    s = synth.vector(n, 4)
    lam = solvers.ritz_lambda_max(lambda x: A @ x, dg, s, 12)
    Dh = np.diag(dg**-0.5)
    B = Dh @ A @ Dh
    v = np.sqrt(dg) * (s / dg)  # start vector of the preconditioned Lanczos: D^{1/2} z0
    V = [v / np.linalg.norm(v)]
    for j in range(11):
        w = B @ V[-1]
        for u in V:
            w -= (u @ w) * u
        for u in V:
            w -= (u @ w) * u
        V.append(w / np.linalg.norm(w))
    V = np.array(V).T
    ref = np.linalg.eigvalsh(V.T @ B @ V)[-1]
    assert abs(lam - ref) < 1e-10 * ref


def _cheb_T(k, t):
    t = np.asarray(t, dtype=float)
    return np.where(np.abs(t) <= 1, np.cos(k * np.arccos(np.clip(t, -1, 1))), np.cosh(k * np.arccosh(np.maximum(np.abs(t), 1))) * np.sign(t) ** k)


@pytest.mark.parametrize("degree", [1, 2, 3, 6])
def test_chebyshev_residual_polynomial_closed_form(degree):
    # r - A x = T_k((theta - lam)/delta) / T_k(theta/delta) r per eigencomponent
    lam_i = np.linspace(0.05, 1.3, 40)
    lam = 1.2
    r = synth.vector(40, 2)
    x = solvers.chebyshev(lambda v: lam_i * v, np.ones(40), r, lam, degree, 20.0)
    a, b = lam / 20, lam
    theta, delta = (a + b) / 2, (b - a) / 2
    R = _cheb_T(degree, (theta - lam_i) / delta) / _cheb_T(degree, theta / delta)
    np.testing.assert_allclose(r - lam_i * x, R * r, rtol=0, atol=1e-13)


def test_chebyshev_degree1_is_damped_jacobi():
    d = np.linspace(1, 3, 20)
    A = lambda v: 2.0 * d * v  # noqa: E731
    r = synth.vector(20, 3)
    lam = 2.4
    x = solvers.chebyshev(A, d, r, lam, 1, 20.0)
    np.testing.assert_allclose(x, r / d * 2.0 / (lam / 20 + lam), rtol=1e-15)


def _solve(p, f_kind=1, tol=1e-12):
    A = oracle.CSR(p)
    b = oracle.rhs(p, f_kind)
    d = A.diagonal()
    s = synth.with_zero_dirichlet(synth.vector(A.n, 0), oracle.constrained_mask_fast(p))
    return A, b, solvers.chebyshev_pcg(A.matvec, d, b, s, rel_tol=tol)


@pytest.mark.parametrize("k,sizes", [(2, (4, 8)), (3, (2, 4)), (1, (8, 16))])
def test_manufactured_l2_rate(k, sizes):
    errs = []
    for n in sizes:
        p = oracle.problem(dim=3, n_cells=(n, n, n), degree=k)
        A, b, res = _solve(p)
        errs.append(oracle.l2_error(p, res.x))
    rate = np.log2(errs[0] / errs[1])
    assert abs(rate - (k + 1)) < 0.15, (errs, rate)


def test_manufactured_l2_rate_2d():
    errs = []
    for n in (8, 16):
        p = oracle.problem(dim=2, n_cells=(n, n), degree=2)
        A, b, res = _solve(p)
        errs.append(oracle.l2_error(p, res.x))
    assert abs(np.log2(errs[0] / errs[1]) - 3) < 0.1


def test_lambda_safety_bounds_true_lambda():
    # O10 pin: 1.2 * Ritz(12) bounds lambda_max(D^{-1} A) from above (Ritz values are interior)
    p = oracle.problem(dim=3, n_cells=(6, 6, 6), degree=2)
    A = oracle.CSR(p)
    d = A.diagonal()
    s = synth.with_zero_dirichlet(synth.vector(A.n, 0), oracle.constrained_mask_fast(p))
    lam = solvers.ritz_lambda_max(A.matvec, d, s, 12)
    Dh = np.diag(d**-0.5)
    true = np.linalg.eigvalsh(Dh @ A.dense() @ Dh)[-1]
    assert lam <= true * (1 + 1e-12)
    assert 1.2 * lam >= true
