"""Pins of the multigrid oracle (oracle/mg.py) against closed
forms and properties the mathematics fixes -- no GPU."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import mg, solvers


def _nodes_1d(k, n_cells, scale=1.0):
    xi = oracle.gll(k)
    return np.array([(c + xi[j]) * scale for c in range(n_cells) for j in range(k)] + [n_cells * scale])


@pytest.mark.parametrize("k", [1, 2, 3, 4, 6, 8])
def test_prolongation_1d_reproduces_the_coarse_space(k):
    # S:621-623 "interpolation of the coarse FE function onto fine support points":
    # every polynomial of degree <= k is in the coarse space, so P x^a(coarse) = x^a(fine)
    P = mg.prolongation_1d(k, 3)
    xc = _nodes_1d(k, 3)
    xf = _nodes_1d(k, 6, 0.5)
    for a in range(k + 1):
        assert np.abs(P @ xc ** a - xf ** a).max() <= 1e-12 * 3.0 ** a
    # partition of unity; a fine node on a coarse node copies it
    assert np.abs(P.sum(axis=1) - 1).max() < 1e-13
    for cc in range(4):
        f, c = 2 * k * cc, k * cc
        np.testing.assert_array_equal(P[f], np.eye(3 * k + 1)[c])


def test_q1_midpoint_rule():
    # S:627 "Q1: fine midpoint value = average of coarse edge endpoints"
    P = mg.prolongation_1d(1, 2)
    np.testing.assert_allclose(P, [[1, 0, 0], [0.5, 0.5, 0], [0, 1, 0], [0, 0.5, 0.5], [0, 0, 1]], atol=1e-15)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_prolongation_3d_reproduces_tensor_polynomials(k):
    nc = (2, 3, 2)
    P = mg.prolongation(k, nc, 3)
    xc = [_nodes_1d(k, n) for n in nc]
    xf = [_nodes_1d(k, 2 * n, 0.5) for n in nc]
    Zc, Yc, Xc = np.meshgrid(xc[2], xc[1], xc[0], indexing="ij")
    Zf, Yf, Xf = np.meshgrid(xf[2], xf[1], xf[0], indexing="ij")
    for (a, b, c) in [(0, 0, 0), (1, 0, 0), (0, 1, 1), (k, k, 0), (k, 1, k)]:
        qc = (Xc ** a * Yc ** b * Zc ** c).ravel()
        qf = (Xf ** a * Yf ** b * Zf ** c).ravel()
        assert np.abs(P @ qc - qf).max() <= 1e-11 * max(1.0, np.abs(qf).max())


@pytest.mark.parametrize("k,nc,upper,coeff", [(1, (8, 4, 4), (1.0, 1.0, 1.0), 1.0),
                                              (2, (4, 2, 2), (1.0, 0.5, 2.0), 2.5),
                                              (3, (4, 2, 2), (1.0, 1.0, 1.0), 1.0)])
def test_galerkin_identity_on_affine_meshes(k, nc, upper, coeff):
    # nested spaces + exact quadrature on affine cells: R A_fine P = A_coarse on the free DoFs
    H = mg.build_hierarchy(3, nc, k, n_levels=2, upper=upper, coeff_value=coeff)
    c, f = H.levels
    Ac = c.A.dense()
    Af = sp.csr_matrix((f.A.val, f.A.col, f.A.rowptr), shape=(f.A.n, f.A.n))
    G = (H.P[1].T @ Af @ H.P[1]).toarray()
    free = ~c.mask
    err = np.abs(G[np.ix_(free, free)] - Ac[np.ix_(free, free)]).max()
    assert err <= 1e-12 * np.abs(Ac).max()
    # constrained rows / columns of the transfer are zero
    assert np.abs(H.P[1].toarray()[f.mask]).max() == 0
    assert np.abs(H.P[1].toarray()[:, c.mask]).max() == 0


@pytest.fixture(scope="module")
def h_q2():
    return mg.build_hierarchy(3, (8, 8, 8), 2, max_coarse_dofs=200)


def test_vcycle_is_linear_and_symmetric(h_q2):
    H = h_q2
    n, mask = H.levels[-1].A.n, H.levels[-1].mask
    rng = np.random.default_rng(3)
    b1, b2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    b1[mask] = 0
    b2[mask] = 0
    v1, v2 = mg.vcycle(H, b1), mg.vcycle(H, b2)
    assert np.abs(mg.vcycle(H, np.zeros(n))).max() == 0.0
    lin = mg.vcycle(H, 2.0 * b1 - 0.5 * b2)
    assert np.linalg.norm(lin - (2.0 * v1 - 0.5 * v2)) <= 1e-12 * np.linalg.norm(lin)
    # same polynomial before and after the coarse correction, exact coarse solve: V = V^T
    assert abs(v1 @ b2 - b1 @ v2) <= 1e-12 * np.linalg.norm(v1) * np.linalg.norm(b2)


def test_one_level_hierarchy_is_the_coarse_solve():
    H = mg.build_hierarchy(3, (2, 2, 2), 2, n_levels=1)
    A = H.levels[0].A
    b = np.random.default_rng(1).uniform(-1, 1, A.n)
    b[H.levels[0].mask] = 0
    x = mg.vcycle(H, b)
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.norm(b)


def test_vcycle_rate_is_small_and_mesh_independent():
    # S:645 / S:664: rates mesh-independent (within 0.03) and well below 0.15 for Chebyshev(6)
    rates = []
    for nc in ((4, 4, 4), (8, 8, 8), (16, 16, 16)):
        H = mg.build_hierarchy(3, nc, 2, max_coarse_dofs=200)
        n, mask = H.levels[-1].A.n, H.levels[-1].mask
        b = np.random.default_rng(5).uniform(-1, 1, n)
        b[mask] = 0
        rates.append(mg.vcycle_rate(H, b, 6))
    assert max(rates) <= 0.15
    assert max(rates) - min(rates) <= 0.03


def test_mg_pcg_converges_in_few_iterations_and_beats_chebyshev_jacobi(h_q2):
    H = h_q2
    A, d, mask = H.levels[-1].A, H.levels[-1].diag, H.levels[-1].mask
    b = oracle.rhs(H.levels[-1].p, 0)
    res = mg.mg_pcg(H, b, 1e-10)
    assert res.iterations <= 8
    x_direct = np.linalg.solve(A.dense(), b)
    assert np.linalg.norm(res.x - x_direct) <= 1e-8 * np.linalg.norm(x_direct)
    s = solvers.chebyshev_pcg(A.matvec, d, b, np.where(mask, 0.0, 1.0), 1e-10)
    assert res.iterations < s.iterations
