"""Unstructured hexahedral-mesh oracle -- TEST INFRASTRUCTURE ONLY.

The paper's method scope includes "general unstructured meshes of quadrilaterals /
hexahedra" with "hanging nodes" handled as constraints inside the matrix-free
gather / scatter (§3.1, §3.5).
This module writes out the plain definition on a mesh given as vertex coordinates
plus, per cell, its 8 vertex numbers in the cell's own lexicographic frame
(local vertex a + 2 b + 4 c sits at reference corner (a, b, c) of [0,1]^3):

  mapping (R21): trilinear, x(xi) = sum_v X_v N_v(xi), N_v the Q1 basis;
  space: continuous Q_k on the GLL support points x(GLL node) of every cell;
  cell matrix: A_c[i][j] = sum_q w_q c(x_q) det J_q (J_q^-T grad phi_i) . (J_q^-T grad phi_j)
      over the Gauss(k+1)^3 points (R1), c constant or R5's 1/(0.05 + 2|x|^2);
  DoF numbering (R21): one DoF per distinct support point, found here by brute force
      on the coordinates (points within 1e-9 of each other are one DoF);
  constraints (R22): a cell-local node either IS a DoF or is a constraint line
      u_local = sum_m w_m u_{dof m} (a hanging node); the global operator is
      A = sum_c P_c^T A_c P_c with P_c the cell's expansion rows;
  Dirichlet (R3): listed DoFs get identity rows and columns.

Everything is brute force: one cell matrix per cell from point-by-point quadrature
with the Lagrange product formula of the pinned 1D rules (oracle.gauss / gll /
lagrange / lagrange_d).  Pins: tests/test_oracle_hex.py (a rotated, renumbered
structured brick equals the structured oracle; linear and quadratic reproduction on
distorted and sheared meshes; rotation and scaling invariance; the 2:1 hanging
interface equals oracle/hanging.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import gauss, gll, lagrange, lagrange_d

_CORNERS = np.array([[v & 1, (v >> 1) & 1, v >> 2] for v in range(8)], dtype=np.float64)


def tables(k: int):
    """1D tables on [0,1]: S[q][i] = l_i(xi_q), D[q][i] = l_i'(xi_q), Gauss weights."""
    xq, wq = gauss(k + 1)
    nodes = gll(k)
    S = np.array([[lagrange(nodes, i, x) for i in range(k + 1)] for x in xq])
    D = np.array([[lagrange_d(nodes, i, x) for i in range(k + 1)] for x in xq])
    return xq, wq, nodes, S, D


def trilinear(Xc: np.ndarray, xi: np.ndarray):
    """x(xi) and J = dx/dxi of the trilinear map of a cell with corner coordinates Xc[8][3]."""
    N = np.ones(8)
    dN = np.ones((8, 3))
    for v in range(8):
        for d in range(3):
            f = xi[d] if _CORNERS[v, d] else 1.0 - xi[d]
            df = 1.0 if _CORNERS[v, d] else -1.0
            N[v] *= f
            for e in range(3):
                dN[v, e] *= df if e == d else f
    x = N @ Xc
    J = Xc.T @ dN  # J[a][e] = d x_a / d xi_e
    return x, J


def coefficient(x: np.ndarray, kind: str, value: float = 1.0) -> float:
    """R5: c(x) = 1 / (0.05 + 2 |x|^2) for 'variable', else the constant."""
    if kind == "variable":
        return 1.0 / (0.05 + 2.0 * float(x @ x))
    return value


def _local_index(k: int):
    n = k + 1
    return [(i % n, (i // n) % n, i // (n * n)) for i in range(n ** 3)]


def cell_matrix(Xc: np.ndarray, k: int, coeff: str = "constant", value: float = 1.0, mass: bool = False):
    """A_c (and the mass matrix M_c with the same quadrature) of one trilinear cell."""
    xq, wq, _, S, D = tables(k)
    n = k + 1
    loc = _local_index(k)
    nv = n ** 3
    A = np.zeros((nv, nv))
    M = np.zeros((nv, nv))
    for q2 in range(n):
        for q1 in range(n):
            for q0 in range(n):
                x, J = trilinear(Xc, np.array([xq[q0], xq[q1], xq[q2]]))
                det = np.linalg.det(J)
                if det <= 0.0:
                    raise FloatingPointError("det J <= 0")
                Jinv = np.linalg.inv(J)
                w = wq[q0] * wq[q1] * wq[q2] * det
                phi = np.array([S[q0, a] * S[q1, b] * S[q2, c] for (a, b, c) in loc])
                gref = np.array([[D[q0, a] * S[q1, b] * S[q2, c], S[q0, a] * D[q1, b] * S[q2, c],
                                  S[q0, a] * S[q1, b] * D[q2, c]] for (a, b, c) in loc])
                grad = gref @ Jinv  # physical gradients: grad_x phi = J^-T grad_xi phi
                A += w * coefficient(x, coeff, value) * grad @ grad.T
                M += w * np.outer(phi, phi)
    return (A, M) if mass else A


def support_points(vertices: np.ndarray, cell_vertices: np.ndarray, k: int) -> np.ndarray:
    """x(GLL node) for every cell and local node: [n_cells][(k+1)^3][3]."""
    nodes = gll(k)
    loc = _local_index(k)
    out = np.zeros((len(cell_vertices), len(loc), 3))
    for c, cv in enumerate(cell_vertices):
        Xc = vertices[cv]
        for i, (a, b, d) in enumerate(loc):
            out[c, i] = trilinear(Xc, np.array([nodes[a], nodes[b], nodes[d]]))[0]
    return out


def number_by_coordinates(points: np.ndarray, tol: float = 1e-9):
    """R21: one DoF per distinct point (first appearance order, cell by cell).
    Returns (cell_dofs [n_cells][nv] int64, dof coordinates [n][3])."""
    flat = points.reshape(-1, 3)
    key = np.round(flat / tol).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty(len(order), dtype=np.int64)
    rank[order] = np.arange(len(order))
    cell_dofs = rank[inv.reshape(-1)].reshape(points.shape[:2])
    return cell_dofs, flat[first[order]]


def assemble(vertices: np.ndarray, cell_vertices: np.ndarray, k: int, cell_dofs: np.ndarray, n_dofs: int,
             lines=None, dirichlet=None, coeff: str = "constant", value: float = 1.0,
             mass: bool = False) -> sp.csr_matrix:
    """A = sum_c P_c^T A_c P_c (R22) with Dirichlet identity rows / columns (R3).

    cell_dofs[c][i] >= 0 is a DoF; -1 - l refers to constraint line l = lines[l], a list
    of (dof, weight) pairs.  Line entries on Dirichlet DoFs contribute nothing (their
    value is zero)."""
    lines = lines or []
    dmask = np.zeros(n_dofs, dtype=bool)
    if dirichlet is not None:
        dmask[np.asarray(dirichlet, dtype=np.int64)] = True
    rows, cols, vals = [], [], []
    for c, cv in enumerate(cell_vertices):
        AM = cell_matrix(vertices[cv], k, coeff, value, mass=mass)
        Ac = AM[1] if mass else AM
        nv = Ac.shape[0]
        P = np.zeros((nv, n_dofs))
        for i in range(nv):
            d = int(cell_dofs[c, i])
            for m, w in ([(d, 1.0)] if d >= 0 else lines[-1 - d]):
                if not dmask[m]:
                    P[i, m] += w
        used = np.nonzero(np.any(P != 0.0, axis=0))[0]
        Pc = P[:, used]
        B = Pc.T @ Ac @ Pc
        r, s = np.meshgrid(used, used, indexing="ij")
        rows.append(r.reshape(-1))
        cols.append(s.reshape(-1))
        vals.append(B.reshape(-1))
    d = np.nonzero(dmask)[0]
    rows.append(d)
    cols.append(d)
    vals.append(np.ones(len(d)))
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n_dofs, n_dofs))


def boundary_dofs(dof_coords: np.ndarray, lower, upper, tol: float = 1e-9) -> np.ndarray:
    """DoFs on the faces of the box [lower, upper] (the meshes here fill a box)."""
    lo, hi = np.asarray(lower), np.asarray(upper)
    on = np.any((np.abs(dof_coords - lo) < tol) | (np.abs(dof_coords - hi) < tol), axis=1)
    return np.nonzero(on)[0]
