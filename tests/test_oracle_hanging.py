"""Pins of the hanging-node oracle (oracle/hanging.py, SURVEY §8(f) f3 restricted to
the two-block 2:1 interface) -- no GPU."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import hanging


@pytest.mark.parametrize("k,nc,nzf", [(1, (2, 2, 1), 2), (2, (2, 2, 2), 2), (3, (2, 1, 1), 1)])
def test_symmetric(k, nc, nzf):
    A = hanging.operator(hanging.build(nc, nzf, k))
    assert abs(A - A.T).max() <= 1e-14 * abs(A).max()


@pytest.mark.parametrize("k,nc,nzf", [(2, (2, 2, 2), 2), (2, (1, 2, 1), 3), (3, (2, 1, 1), 1)])
def test_exact_on_the_polynomial_space(k, nc, nzf):
    # u = x(1-x)y(1-y)z(1-z) is in Q_k of both blocks, vanishes on the boundary and meets
    # the hanging constraints exactly, so A u = M (-lap u) on every free row
    T = hanging.build(nc, nzf, k)
    x, y, z = hanging.node_coords(T).T
    u = x * (1 - x) * y * (1 - y) * z * (1 - z)
    f = 2 * (y * (1 - y) * z * (1 - z) + x * (1 - x) * z * (1 - z) + x * (1 - x) * y * (1 - y))
    r = hanging.operator(T) @ u - hanging.operator_unconstrained(T, 1) @ f
    assert np.abs(r[~T.mask]).max() <= 1e-13 * np.abs(hanging.operator(T) @ u).max()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_constants_in_the_kernel_without_constraints(k):
    T = hanging.build((2, 1, 1), 2, k)
    A = hanging.operator_unconstrained(T)
    assert np.abs(A @ np.ones(T.n)).max() <= 1e-13 * abs(A).max()


@pytest.mark.parametrize("k", [1, 2])
def test_manufactured_convergence_on_the_nonconforming_mesh(k):
    errs = []
    for n in (4, 8):
        T = hanging.build((n, n, n // 2), n // 2, k)
        u = spla.spsolve(hanging.operator(T).tocsc(), hanging.load(T, 1))
        errs.append(hanging.error(T, u))
    assert abs(np.log2(errs[0] / errs[1]) - (k + 1)) < 0.2
