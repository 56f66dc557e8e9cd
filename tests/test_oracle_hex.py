"""Pins of the unstructured-hex oracle (oracle/hex.py).

Each pin ties oracle.hex to something other than itself:
  * a structured brick fed as an unstructured mesh -- cells in random local frames
    (24 cube rotations), vertices renumbered -- equals the structured oracle
    (oracle.CSR, pinned by test_oracle_operator.py) after matching DoFs by
    coordinates, for constant and variable coefficient (a transposed J, a wrong
    frame rotation or a dropped coefficient fails it);
  * physical linears on a jittered (genuinely trilinear) mesh: A u = 0 on interior
    rows, A 1 = 0 without Dirichlet (Galerkin exactness: the integrand
    c . adj(J)^T grad phi is a polynomial Gauss(k+1) integrates exactly);
  * quadratics on a sheared (affine, non-orthogonal) mesh: A u = -tr(H) M 1 on
    interior rows (exact quadrature for affine cells; pins the J^-T terms that a
    box never exercises);
  * invariance under a rotation about the origin (variable coefficient too, |x| is
    preserved) and scaling A(s X) = s A(X) for constant coefficient;
  * the 2:1 hanging interface built from constraint lines equals oracle/hanging.py
    (pinned by test_oracle_hanging.py).
"""
import numpy as np
import pytest

import oracle
from oracle import hex as ohex
from tests import _hexmesh as hm


def _structured_coords(n_cells, k, lower, upper):
    nodes = oracle.gll(k)
    ax = []
    for e in range(3):
        h = (upper[e] - lower[e]) / n_cells[e]
        pts = [lower[e] + h * (c + nodes[i]) for c in range(n_cells[e]) for i in range(k + (c == n_cells[e] - 1))]
        ax.append(np.array(pts))
    Z, Y, X = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.stack([X.reshape(-1), Y.reshape(-1), Z.reshape(-1)], axis=1)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("coeff", ["constant", "variable"])
def test_rotated_brick_equals_structured_oracle(k, coeff):
    n_cells, lower, upper = (2, 3, 2), (-0.3, 0.1, 0.0), (0.9, 1.0, 0.7)
    m = hm.conforming(n_cells, k, lower, upper, jitter=0.0, seed=k)
    A = hm.oracle_matrix(m, coeff=coeff, value=1.7).toarray()
    p = oracle.problem(dim=3, n_cells=n_cells, degree=k, lower=lower, upper=upper,
                       coeff_kind=1 if coeff == "variable" else 0, coeff_value=1.7)
    S = oracle.CSR(p).dense()
    perm = hm.match(m["coords"], _structured_coords(n_cells, k, lower, upper))
    assert m["n_dofs"] == S.shape[0]
    B = S[np.ix_(perm, perm)]
    assert np.abs(A - B).max() <= 1e-13 * np.abs(B).max()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_linears_on_jittered_mesh(k):
    m = hm.conforming((3, 2, 2), k, jitter=0.25, seed=7 + k)
    A = hm.oracle_matrix(m, dirichlet=False)
    one = np.ones(m["n_dofs"])
    assert np.abs(A @ one).max() <= 1e-13 * abs(A).max()
    u = m["coords"] @ np.array([0.3, -1.1, 0.7]) + 0.4
    interior = np.setdiff1d(np.arange(m["n_dofs"]), m["dirichlet"])
    assert np.abs((A @ u)[interior]).max() <= 1e-12 * abs(A).max()
    # not a vacuous check: the boundary rows carry the flux
    assert np.abs((A @ u)[m["dirichlet"]]).max() > 1e-3
    # symmetric positive definite with Dirichlet rows
    Ad = hm.oracle_matrix(m).toarray()
    assert np.abs(Ad - Ad.T).max() <= 1e-14 * np.abs(Ad).max()
    assert np.linalg.eigvalsh(Ad).min() > 0


@pytest.mark.parametrize("k", [1, 2, 3])
def test_variable_coefficient_energy_of_linears_on_jittered_mesh(k):
    # u_a^T A u_b = delta_ab int c dx for the physical linears u_a = x_a under Neumann (the
    # jitter moves interior vertices only, so the mesh covers the unit cube exactly): G is a
    # multiple of the identity to rounding, its diagonal converges to the mesh-free integral
    # of c (tests/test_oracle_operator.py::_integral_of_c_unit_cube)
    from tests.test_oracle_operator import _integral_of_c_unit_cube

    Ic = _integral_of_c_unit_cube()
    errs = []
    for n in (2, 6):
        m = hm.conforming((n, n, n), k, jitter=0.25, seed=11 + k)
        A = hm.oracle_matrix(m, coeff="variable", dirichlet=False)
        X = m["coords"]
        G = np.array([[X[:, a] @ (A @ X[:, b]) for b in range(3)] for a in range(3)])
        assert np.abs(G - G[0, 0] * np.eye(3)).max() <= 1e-13 * Ic
        errs.append(abs(G[0, 0] - Ic) / Ic)
    assert errs[1] <= errs[0] / 9  # converging (at least h^2 over a 3x refinement)
    assert errs[1] <= {1: 3e-4, 2: 3e-5, 3: 2e-6}[k]  # measured 1.6e-4, 1.3e-5, 6.3e-7


@pytest.mark.parametrize("k", [2, 3])
def test_quadratics_on_sheared_mesh(k):
    m = hm.conforming((2, 2, 2), k, jitter=0.0, seed=3)
    B = np.array([[1.0, 0.35, -0.2], [0.0, 0.9, 0.25], [0.1, 0.0, 1.1]])
    m["vertices"] = m["vertices"] @ B.T
    m["coords"] = m["coords"] @ B.T
    A = hm.oracle_matrix(m, dirichlet=False)
    M = hm.oracle_matrix(m, dirichlet=False, mass=True)
    H = np.array([[2.0, 0.5, -0.3], [0.5, -1.0, 0.8], [-0.3, 0.8, 0.6]])
    x = m["coords"]
    u = 0.5 * np.einsum("ni,ij,nj->n", x, H, x) + x @ np.array([0.2, 0.1, -0.4])
    interior = np.setdiff1d(np.arange(m["n_dofs"]), m["dirichlet"])
    lhs = (A @ u)[interior]
    rhs = -np.trace(H) * (M @ np.ones(m["n_dofs"]))[interior]
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()


def test_rotation_and_scaling_invariance():
    m = hm.conforming((2, 2, 3), 2, lower=(-0.5, -0.4, -0.6), upper=(0.5, 0.6, 0.4), jitter=0.2, seed=11)
    th = 0.7
    Q = np.array([[np.cos(th), -np.sin(th), 0.0], [np.sin(th), np.cos(th), 0.0], [0.0, 0.0, 1.0]])
    Q = Q @ np.array([[1.0, 0.0, 0.0], [0.0, np.cos(0.4), -np.sin(0.4)], [0.0, np.sin(0.4), np.cos(0.4)]])
    for coeff in ("constant", "variable"):
        A0 = hm.oracle_matrix(m, coeff=coeff).toarray()
        r = dict(m, vertices=m["vertices"] @ Q.T)
        A1 = hm.oracle_matrix(r, coeff=coeff).toarray()
        assert np.abs(A1 - A0).max() <= 1e-13 * np.abs(A0).max()
    s = 2.5
    A0 = hm.oracle_matrix(m, dirichlet=False).toarray()
    A2 = hm.oracle_matrix(dict(m, vertices=s * m["vertices"]), dirichlet=False).toarray()
    assert np.abs(A2 - s * A0).max() <= 1e-13 * np.abs(A2).max()


@pytest.mark.parametrize("k", [1, 2, 3])
def test_hanging_interface_equals_two_block_oracle(k):
    from oracle import hanging

    n_cells, nzf = (2, 1, 1), 2
    m = hm.two_block(n_cells, nzf, k)
    T = hanging.build(n_cells, nzf, k)
    assert m["n_dofs"] == T.n
    A = hm.oracle_matrix(m).toarray()
    H = hanging.operator(T).toarray()
    perm = hm.match(m["coords"], hanging.node_coords(T))
    B = H[np.ix_(perm, perm)]
    assert np.abs(A - B).max() <= 1e-13 * np.abs(B).max()
    assert len(m["lines"]) > 0


def test_degenerate_cell_is_rejected():
    V, C = np.eye(8, 3), np.arange(8, dtype=np.int32)[None, :]
    with pytest.raises(FloatingPointError):
        ohex.cell_matrix(V[C[0]], 1)
