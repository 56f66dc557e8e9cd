"""Exact-integration helpers for oracle pins (test-only, independent of the
oracle's quadrature): 1D Lagrange polynomials on the GLL nodes are built from
their roots in numpy's Legendre basis and integrated exactly."""
import numpy as np
from numpy.polynomial import Legendre
from numpy.polynomial import legendre as L


def gll_ref(k):
    if k == 1:
        return np.array([0.0, 1.0])
    r = np.sort(L.Legendre.basis(k).deriv().roots())
    return 0.5 * (1 + np.concatenate([[-1.0], r, [1.0]]))


def lagrange_polys(nodes):
    polys = []
    for i, xi in enumerate(nodes):
        others = np.delete(nodes, i)
        p = Legendre.fromroots(others, domain=[0, 1])  # Legendre basis: well conditioned to k = 8
        polys.append(p / p(xi))
    return polys


def exact_1d(k, h=1.0):
    """1D element stiffness K and mass M on [0, h] by exact integration."""
    ps = lagrange_polys(gll_ref(k))
    n = k + 1
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            pk = (ps[i].deriv() * ps[j].deriv()).integ()
            pm = (ps[i] * ps[j]).integ()
            K[i, j] = (pk(1.0) - pk(0.0)) / h
            M[i, j] = (pm(1.0) - pm(0.0)) * h
    return K, M


def exact_cell(k, h, dim):
    """Affine box cell with sides h[e], c = 1: sum_e K_e (x) M_others, index (z,y,x)."""
    KM = [exact_1d(k, h[e]) for e in range(dim)]
    A = 0
    for e in range(dim):
        T = np.ones((1, 1))
        for d in reversed(range(dim)):  # slowest (z) first for np.kron
            T = np.kron(T, KM[d][0] if d == e else KM[d][1])
        A = A + T
    return A


def integral_of_basis_1d(k, h, n_cells):
    """int phi_m over [0, n_cells h] for every global 1D node m."""
    ps = lagrange_polys(gll_ref(k))
    w = np.array([(p.integ()(1.0) - p.integ()(0.0)) * h for p in ps])
    out = np.zeros(k * n_cells + 1)
    for c in range(n_cells):
        out[k * c:k * c + k + 1] += w
    return out
