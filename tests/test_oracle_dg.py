"""Pins of the DG-SIP oracle (oracle/dg.py) -- no GPU:
symmetry and positivity, the continuous subspace (E^T A_DG E = A_CG on functions
that vanish on the boundary), a Kronecker-sum identity against an independent 1D
SIP assembly, and the O(h^{k+1}) L2 convergence of the manufactured solution."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle
from oracle import dg


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_symmetric_positive_definite(k):
    A = dg.assemble((2, 2, 1), k).toarray()
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0.0


@pytest.mark.parametrize("k,nc", [(1, (3, 2, 2)), (2, (2, 2, 2)), (3, (2, 1, 2))])
def test_continuous_subspace_is_the_cg_operator(k, nc):
    # for continuous u, v that vanish on the boundary every face term is zero, so
    # E^T A_DG E equals the (pinned) CG stiffness matrix on the free DoFs
    A = dg.assemble(nc, k).toarray()
    p = oracle.problem(dim=3, n_cells=nc, degree=k)
    Acg = oracle.CSR(p).dense()
    free = ~oracle.constrained_mask_fast(p)
    N = k + 1
    E = np.zeros((A.shape[0], Acg.shape[0]))
    for cell in range(nc[0] * nc[1] * nc[2]):
        for i, g in enumerate(oracle.cell_dofs(p, cell)):
            E[cell * N ** 3 + i, g] = 1.0
    G = E.T @ A @ E
    assert np.abs(G[np.ix_(free, free)] - Acg[np.ix_(free, free)]).max() <= 1e-12 * np.abs(Acg).max()


def _sip_1d(n, k, h):
    """Independent 1D SIP: cell stiffness from Gauss quadrature of l_i' l_j', point terms
    at interior / boundary points; mass blocks h * int l_i l_j."""
    N = k + 1
    nodes = oracle.gll(k)
    xq, wq = oracle.gauss(N)
    d = np.array([[oracle.lagrange_d(nodes, i, x) for x in xq] for i in range(N)])
    v = np.array([[oracle.lagrange(nodes, i, x) for x in xq] for i in range(N)])
    Kc = (d * wq) @ d.T / h
    Mc = (v * wq) @ v.T * h
    val0 = np.array([oracle.lagrange(nodes, i, 0.0) for i in range(N)])
    val1 = np.array([oracle.lagrange(nodes, i, 1.0) for i in range(N)])
    der0 = np.array([oracle.lagrange_d(nodes, i, 0.0) for i in range(N)]) / h
    der1 = np.array([oracle.lagrange_d(nodes, i, 1.0) for i in range(N)]) / h
    sig = 2.0 * (k + 1) ** 2 / h
    A = np.zeros((n * N, n * N))
    M = np.zeros((n * N, n * N))
    for c in range(n):
        s = slice(c * N, (c + 1) * N)
        A[s, s] += Kc
        M[s, s] += Mc
    for c in range(n - 1):  # point between cell c (its 1) and c + 1 (its 0), n = +x
        J = np.zeros(n * N)
        Dv = np.zeros(n * N)
        J[c * N:(c + 1) * N] += val1
        J[(c + 1) * N:(c + 2) * N] -= val0
        Dv[c * N:(c + 1) * N] += 0.5 * der1
        Dv[(c + 1) * N:(c + 2) * N] += 0.5 * der0
        A += -np.outer(J, Dv) - np.outer(Dv, J) + sig * np.outer(J, J)
    for c, val, der, sgn in ((0, val0, der0, -1.0), (n - 1, val1, der1, 1.0)):  # boundary points
        V = np.zeros(n * N)
        D = np.zeros(n * N)
        V[c * N:(c + 1) * N] = val
        D[c * N:(c + 1) * N] = sgn * der
        A += -np.outer(V, D) - np.outer(D, V) + sig * np.outer(V, V)
    return A, M


@pytest.mark.parametrize("k,nc,upper", [(1, (3, 2, 2), (1.0, 1.0, 1.0)), (2, (2, 3, 2), (1.0, 0.5, 2.0)),
                                        (4, (2, 1, 1), (1.0, 1.0, 1.0))])
def test_kronecker_sum_identity(k, nc, upper):
    # on axis-aligned cells every face integral factors: A = A1x (x) M1y (x) M1z + ...
    A = dg.assemble(nc, k, upper=upper).toarray()
    N = k + 1
    h = [upper[e] / nc[e] for e in range(3)]
    A1 = [_sip_1d(nc[e], k, h[e]) for e in range(3)]
    Kr = (np.kron(A1[2][1], np.kron(A1[1][1], A1[0][0])) + np.kron(A1[2][1], np.kron(A1[1][0], A1[0][1]))
          + np.kron(A1[2][0], np.kron(A1[1][1], A1[0][1])))
    # DG index (cell, local) -> Kronecker index (gz, gy, gx) with g_e = c_e N + i_e
    n1 = [nc[e] * N for e in range(3)]
    perm = np.zeros(A.shape[0], dtype=int)
    for cz in range(nc[2]):
        for cy in range(nc[1]):
            for cx in range(nc[0]):
                cell = cx + nc[0] * (cy + nc[1] * cz)
                for i in range(N ** 3):
                    ix, iy, iz = i % N, (i // N) % N, i // (N * N)
                    gx, gy, gz = cx * N + ix, cy * N + iy, cz * N + iz
                    perm[cell * N ** 3 + i] = gx + n1[0] * (gy + n1[1] * gz)
    assert np.abs(A - Kr[np.ix_(perm, perm)]).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("k", [1, 2])
def test_manufactured_convergence(k):
    f = lambda x, y, z: 3 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)  # noqa: E731
    ex = lambda x, y, z: np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)  # noqa: E731
    errs = []
    for n in (4, 8):
        A = dg.assemble((n, n, n), k)
        u = spla.spsolve(A.tocsc(), dg.rhs((n, n, n), k, f))
        errs.append(dg.l2_error((n, n, n), k, u, ex))
    assert abs(np.log2(errs[0] / errs[1]) - (k + 1)) < 0.15
