"""Pins for the oracle's element and global operator (O3-O8, O12).

Each test ties the oracle to something other than itself: the SPEC's worked
example, exact polynomial integration with numpy.polynomial, closed
forms of the Q1 stencils and spectrum, harmonic-polynomial identities,
Neumann kernel / volume / symmetry invariants and convergence theory."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests import _exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_q1_unit_square_cell_matrix_spec_example():
    g = json.load(open(os.path.join(GOLDEN, "q1_unit_square_cell_matrix.json")))
    p = oracle.problem(dim=2, n_cells=(1, 1), degree=1, dirichlet=0)
    A = oracle.cell_matrix(p, 0)
    np.testing.assert_allclose(A, np.array(g["matrix_times_6"]) * g["scale"], rtol=0, atol=g["tol"])


def test_q1_unit_cube_cell_closed_form():
    # 3D Q1 unit cube x12: diag 4, axis neighbour 0, face diagonal -1, body diagonal -1
    p = oracle.problem(dim=3, n_cells=(1, 1, 1), degree=1, dirichlet=0)
    A = 12 * oracle.cell_matrix(p, 0)
    for i in range(8):
        for j in range(8):
            hd = bin(i ^ j).count("1")
            assert abs(A[i, j] - {0: 4, 1: 0, 2: -1, 3: -1}[hd]) < 1e-13


def test_q2_1d_element_closed_form():
    g = json.load(open(os.path.join(GOLDEN, "q2_1d_element.json")))
    for h in (1.0, 0.25):
        p = oracle.problem(dim=1, n_cells=(1,), degree=2, upper=(h,), dirichlet=0)
        A, M = oracle.cell_matrix(p, 0, mass=True)
        np.testing.assert_allclose(A * 3 * h, g["K_times_3h"], atol=1e-13)
        np.testing.assert_allclose(M * 30 / h, g["M_times_30_over_h"], atol=1e-13)
        p1 = oracle.problem(dim=1, n_cells=(1,), degree=1, upper=(h,), dirichlet=0)
        A1, M1 = oracle.cell_matrix(p1, 0, mass=True)
        np.testing.assert_allclose(A1 * h, g["Q1_K_times_h"], atol=1e-14)
        np.testing.assert_allclose(M1 * 6 / h, g["Q1_M_times_6_over_h"], atol=1e-14)


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 3), (2, 6), (2, 8), (3, 1), (3, 2), (3, 3), (3, 4), (3, 5)])
def test_affine_cell_matches_exact_integration(dim, k):
    # brute force (exact polynomial integration, no quadrature) on an anisotropic box cell
    h = [0.5, 0.25, 0.125][:dim]
    nc = [2, 4, 8][:dim]
    p = oracle.problem(dim=dim, n_cells=nc, degree=k, dirichlet=0)
    A = oracle.cell_matrix(p, 0)
    ref = _exact.exact_cell(k, h, dim)
    assert np.abs(A - ref).max() <= 1e-12 * np.abs(ref).max()


def test_q1_global_stencils():
    # 2D Q1 interior stencil (1/3)[8; -1 x 8]; 3D Q1: 8h/3, axis 0, edge -h/6, corner -h/12
    p = oracle.problem(dim=2, n_cells=(4, 4), degree=1, dirichlet=0)
    D = oracle.CSR(p, dirichlet=False).dense()
    row = D[2 * 5 + 2].reshape(5, 5)
    np.testing.assert_allclose(row[1:4, 1:4], np.array([[-1, -1, -1], [-1, 8, -1], [-1, -1, -1]]) / 3, atol=1e-14)
    n = 4
    h = 1.0 / n
    p = oracle.problem(dim=3, n_cells=(n, n, n), degree=1, dirichlet=0)
    D = oracle.CSR(p, dirichlet=False).dense()
    g = (2 * 5 + 2) * 5 + 2
    r = D[g].reshape(5, 5, 5)[1:4, 1:4, 1:4]
    for dz in range(3):
        for dy in range(3):
            for dx in range(3):
                m = abs(dz - 1) + abs(dy - 1) + abs(dx - 1)
                assert abs(r[dz, dy, dx] - {0: 8 * h / 3, 1: 0, 2: -h / 6, 3: -h / 12}[m]) < 1e-14


def test_q1_4x4_spectrum_closed_form():
    g = json.load(open(os.path.join(GOLDEN, "q1_2d_4x4_spectrum.json")))
    p = oracle.problem(dim=2, n_cells=(4, 4), degree=1)
    D = oracle.CSR(p).dense()
    free = ~oracle.constrained_mask(p)
    ev = np.linalg.eigvalsh(D[np.ix_(free, free)])
    t = np.array(g["theta_over_pi"]) * np.pi
    ref = np.sort([8 / 3 - (2 / 3) * (np.cos(a) + np.cos(b)) - (4 / 3) * np.cos(a) * np.cos(b) for a in t for b in t])
    np.testing.assert_allclose(ev, ref, atol=g["tol"])
    distinct = np.unique(np.round(ev, 10))
    np.testing.assert_allclose(distinct, g["distinct_eigenvalues"], atol=1e-10)


def test_dirichlet_identity_rows():
    p = oracle.problem(dim=3, n_cells=(2, 3, 2), degree=2)
    A = oracle.CSR(p)
    D = A.dense()
    m = oracle.constrained_mask(p)
    assert np.array_equal(m, oracle.constrained_mask_fast(p))
    np.testing.assert_array_equal(D[np.ix_(m, m)], np.eye(m.sum()))
    assert np.all(D[np.ix_(m, ~m)] == 0) and np.all(D[np.ix_(~m, m)] == 0)
    np.testing.assert_array_equal(A.diagonal()[m], 1.0)


@pytest.mark.parametrize("geom,coeff_kind", [(0, 0), (1, 0), (1, 1), (0, 1)])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_neumann_kernel_symmetry(geom, coeff_kind, k):
    # constants in the kernel of the Neumann matrix; symmetry
    p = oracle.problem(dim=3, n_cells=(3, 2, 2), degree=k, geom=geom, coeff_kind=coeff_kind, dirichlet=0)
    A = oracle.CSR(p, dirichlet=False)
    D = A.dense()
    one = np.ones(A.n)
    assert np.abs(A @ one).max() <= 1e-14 * np.abs(D).sum(1).max()
    assert np.abs(D - D.T).max() <= 1e-14 * np.abs(D).max()


@pytest.mark.parametrize("geom", [0, 1])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_mass_sums_to_volume(geom, k):
    # mass-matrix entries sum to |Omega| = 1; Phi maps the unit cube onto itself (R4)
    p = oracle.problem(dim=3, n_cells=(3, 3, 2), degree=k, geom=geom, dirichlet=0)
    M = oracle.CSR(p, which=1, dirichlet=False)
    assert abs(M.val.sum() - 1.0) < 1e-13


def _node_coords(p, physical=False):
    """brick (or Phi-mapped) coordinates of every global node, written out in numpy."""
    k = p.degree
    N = [k * p.nc[e] + 1 for e in range(p.dim)]
    axes = []
    for e in range(p.dim):
        h = (p.hi[e] - p.lo[e]) / p.nc[e]
        x1 = np.zeros(N[e])
        g = _exact.gll_ref(k)
        for c in range(p.nc[e]):
            x1[k * c:k * c + k + 1] = p.lo[e] + h * (c + g)
        axes.append(x1)
    grids = np.meshgrid(*axes[::-1], indexing="ij")[::-1]  # x fastest
    X = np.stack([gg.reshape(-1) for gg in grids], axis=1)
    if physical and p.geom == 1:
        t = (X - np.array(p.lo[:p.dim])) / (np.array(p.hi[:p.dim]) - np.array(p.lo[:p.dim]))
        s = np.prod(np.sin(np.pi * t), axis=1)
        X = X + p.eps * (np.array(p.hi[:p.dim]) - np.array(p.lo[:p.dim]))[None, :] * s[:, None]
    return X


def _interior(p):
    X = _node_coords(p)
    lo = np.array(p.lo[:p.dim])
    hi = np.array(p.hi[:p.dim])
    return np.all((X > lo + 1e-12) & (X < hi - 1e-12), axis=1)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_affine_harmonic_polynomials_in_kernel(k):
    p = oracle.problem(dim=3, n_cells=(3, 3, 3), degree=k, upper=(1.0, 0.75, 1.5), dirichlet=0)
    A = oracle.CSR(p, dirichlet=False)
    X = _node_coords(p)
    x, y, z = X.T
    inner = _interior(p)
    polys = [x, y - 2 * z, x * y * z, x * x - y * y]
    if k >= 3:
        polys.append(x * x * y - y**3 / 3)
    for u in polys:
        r = A @ u
        scale = np.abs(A.val).max() * np.abs(u).max()
        assert np.abs(r[inner]).max() <= 1e-13 * scale


@pytest.mark.parametrize("k", [2, 3, 4])
def test_affine_r2_identity(k):
    # (A I(r^2))_i = -2 d int phi_i for interior i (Delta r^2 = 2d); int phi_i by exact integration
    nc = (3, 2, 4)
    up = (1.0, 0.5, 2.0)
    p = oracle.problem(dim=3, n_cells=nc, degree=k, upper=up, dirichlet=0)
    A = oracle.CSR(p, dirichlet=False)
    X = _node_coords(p)
    u = (X**2).sum(1)
    W = [_exact.integral_of_basis_1d(k, up[e] / nc[e], nc[e]) for e in range(3)]
    intphi = np.einsum("k,j,i->kji", W[2], W[1], W[0]).reshape(-1)
    inner = _interior(p)
    r = A @ u
    scale = np.abs(A.dense()).sum(1).max() * np.abs(u).max()  # |A|_inf |u|_inf (R11)
    np.testing.assert_allclose(r[inner], -6 * intphi[inner], rtol=1e-12, atol=1e-14 * scale)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_deformed_linears_reproduced(k):
    # isoparametric: physical linears lie in the FE space; interior rows of A I(a + b.x) vanish (R10)
    p = oracle.problem(dim=3, n_cells=(3, 3, 3), degree=k, geom=1, eps=0.1, dirichlet=0)
    A = oracle.CSR(p, dirichlet=False)
    X = _node_coords(p, physical=True)
    u = 0.3 + X @ np.array([1.0, -2.0, 0.5])
    r = A @ u
    inner = _interior(p)
    assert np.abs(r[inner]).max() <= 1e-13 * np.abs(A.val).max() * np.abs(u).max()


def _integral_of_c_unit_cube(m=8, q=16):
    """int_[0,1]^3 c(x) dx for R5's c(x) = 1/(0.05 + 2|x|^2), by a tensor Gauss rule on m^3
    sub-boxes (numpy leggauss) -- no mesh, no mapping, nothing from the oracle; converged to
    1e-16 at (8, 16) (equal to the (4, 16) and (12, 16) rules)."""
    from numpy.polynomial.legendre import leggauss

    x, w = leggauss(q)
    pts = (np.arange(m)[:, None] + (x[None, :] + 1) / 2).ravel() / m
    ws = np.tile(w / 2, m) / m
    X, Y, Z = np.meshgrid(pts, pts, pts, indexing="ij", sparse=True)
    W = ws[:, None, None] * ws[None, :, None] * ws[None, None, :]
    return float((W / (0.05 + 2 * (X * X + Y * Y + Z * Z))).sum())


# |G00 - int c| / int c at n = 8 cells per direction, with margin over the measured
# quadrature errors 1.9e-5, 1.6e-6, 7.6e-8, 2.0e-9 (k = 1..4)
_ENERGY_TOL_N8 = {1: 1e-4, 2: 1e-5, 3: 1e-6, 4: 2e-8}


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_deformed_variable_coefficient_energy_of_linears(k):
    # Pins the curved, variable-coefficient operator (R4, R5) beyond its invariants.  A physical
    # linear u_a = x_a lies in the isoparametric space, its gradient is e_a, so
    #   u_a^T A u_b = int c grad(x_a) . grad(x_b) dx = delta_ab int c dx   (Neumann).
    # The discrete sum sum_q c(x_q) w_q |det J_q| (J^-T J^T e_a).(J^-T J^T e_b) is delta_ab times
    # ONE quadrature of int c, so G = [u_a^T A u_b] must be a multiple of the identity to
    # rounding (a transposed J^-1 J^-T, a wrong metric entry or a missing symmetric term breaks
    # that), and its diagonal must converge to the mesh-free integral of c (a missing |det J|,
    # c at the reference point instead of x_q, or a wrong Gauss weight breaks that).
    Ic = _integral_of_c_unit_cube()
    errs = []
    for n in (2, 8):
        p = oracle.problem(dim=3, n_cells=(n, n, n), degree=k, geom=1, eps=0.1, coeff_kind=1, dirichlet=0)
        A = oracle.CSR(p, dirichlet=False)
        X = _node_coords(p, physical=True)
        G = np.array([[X[:, a] @ (A @ X[:, b]) for b in range(3)] for a in range(3)])
        assert np.abs(G - G[0, 0] * np.eye(3)).max() <= 1e-13 * Ic
        errs.append(abs(G[0, 0] - Ic) / Ic)
    assert errs[1] <= _ENERGY_TOL_N8[k]
    assert errs[1] <= errs[0] / 16  # converging (at least h^2 over a 4x refinement)


def test_deformed_jacobian_positive():
    p = oracle.problem(dim=3, n_cells=(2, 2, 2), degree=3, geom=1, eps=0.1)
    for c in range(8):
        oracle.cell_matrix(p, c)  # raises if det J <= 0
    bad = oracle.problem(dim=3, n_cells=(2, 2, 2), degree=3, geom=1, eps=2.0)
    with pytest.raises(FloatingPointError):
        for c in range(8):
            oracle.cell_matrix(bad, c)


@pytest.mark.parametrize("dim,nc,k", [(2, (4, 4), 1), (2, (3, 5), 4), (3, (4, 3, 2), 2), (3, (2, 2, 3), 5), (3, (4, 4, 4), 4)])
def test_kron_matches_csr(dim, nc, k):
    up = (1.0, 0.7, 1.3)[:dim]
    p = oracle.problem(dim=dim, n_cells=nc, degree=k, upper=up, coeff_value=1.7)
    A = oracle.CSR(p)
    for seed in (1, 2):
        x = synth.vector(A.n, seed)
        y1 = A @ x
        y2 = oracle.kron_apply(p, x)
        assert np.linalg.norm(y1 - y2) <= 1e-14 * np.linalg.norm(y1)


@pytest.mark.parametrize("geom,coeff_kind,k", [(0, 0, 3), (1, 1, 2), (1, 1, 3), (1, 0, 4)])
def test_apply_rows_matches_csr(geom, coeff_kind, k):
    p = oracle.problem(dim=3, n_cells=(3, 2, 4), degree=k, geom=geom, coeff_kind=coeff_kind)
    A = oracle.CSR(p)
    x = synth.vector(A.n, 3)
    y = A @ x
    rows = np.arange(0, A.n, 7)
    np.testing.assert_allclose(oracle.apply_rows(p, rows, x), y[rows], rtol=0, atol=1e-13 * np.abs(y).max())


def test_rhs_constant_sums_to_free_integral():
    # f = 1, Neumann: sum_i b_i = |Omega| (partition of unity); affine and deformed
    for geom in (0, 1):
        p = oracle.problem(dim=3, n_cells=(3, 3, 3), degree=3, geom=geom, dirichlet=0)
        assert abs(oracle.rhs(p, 0).sum() - 1.0) < 1e-13


@pytest.mark.parametrize("geom,coeff_kind,k", [(0, 0, 1), (0, 0, 3), (1, 1, 2), (1, 1, 4)])
def test_csr_diagonal_equals_dense_diagonal_on_free_rows(geom, coeff_kind, k):
    # CSR.diagonal() (the a9 reference of the GPU diagonal) is the diagonal of the assembled
    # matrix itself (Eq. (1)): compare with diag(dense()) on the free rows, where the
    # entries come from the quadrature, and on the constrained rows (identity, R3)
    p = oracle.problem(dim=3, n_cells=(3, 2, 2), degree=k, geom=geom, coeff_kind=coeff_kind)
    A = oracle.CSR(p)
    m = oracle.constrained_mask_fast(p)
    d, D = A.diagonal(), np.diag(A.dense())
    assert (~m).sum() > 0
    np.testing.assert_array_equal(d[~m], D[~m])
    np.testing.assert_array_equal(d[m], 1.0)
    assert np.all(d[~m] > 0)
