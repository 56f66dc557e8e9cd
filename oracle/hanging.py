"""Hanging-node oracle (restricted) -- TEST INFRASTRUCTURE ONLY.

The simplest adaptive mesh with hanging nodes (§3.5: "hanging
nodes ... constraints"): the box [lo, hi] cut at z = z_mid into a
coarse lower block of (nx, ny, nzc) cells and a fine upper block refined once more,
(2 nx, 2 ny, nzf) cells.  On the interface every coarse cell face meets four fine
faces; the fine interface nodes that are not coarse nodes hang.  Continuity makes
the fine interface values the coarse face function interpolated at the fine
nodes: u_f(interface) = (P_y (x) P_x) u_c(interface), the 2D case of the
multigrid prolongation (oracle/mg.py, pinned).  Global DoFs (R20):
every node of the coarse grid, then the fine grid's nodes above the interface
plane (x-fastest, plane by plane); the fine interface plane is eliminated.

  A = A_c (extended by zeros) + E^T A_f E,

A_c the coarse block's operator (Dirichlet identity on its x, y and bottom faces,
the interface face natural), A_f the fine block's (identity on x, y and top
faces), E: global -> fine-grid vector (identity on the fine nodes above the
interface, the 2D prolongation of the coarse interface plane below it, zero rows
on the fine interface boundary lines -- they are Dirichlet nodes, zero under the
identity convention).  The same E carries the right-hand side and the mass matrix.
Pins: tests/test_oracle_hanging.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import CSR, constrained_mask_fast, l2_error, problem, rhs
from .mg import prolongation


@dataclass
class TwoBlock:
    pc: object
    pf: object
    E: sp.csr_matrix      # fine grid <- global
    nc_dofs: int          # coarse grid DoFs (global prefix)
    n: int                # global DoFs
    mask: np.ndarray      # global Dirichlet DoFs


def build(n_cells=(2, 2, 1), nzf=2, k=2, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0), z_mid=0.5) -> TwoBlock:
    nx, ny, nzc = n_cells
    pc = problem(dim=3, n_cells=(nx, ny, nzc), degree=k, lower=lower, upper=(upper[0], upper[1], z_mid),
                 dirichlet=0b011111)
    pf = problem(dim=3, n_cells=(2 * nx, 2 * ny, nzf), degree=k, lower=(lower[0], lower[1], z_mid), upper=upper,
                 dirichlet=0b101111)
    Nc = [k * nx + 1, k * ny + 1, k * nzc + 1]
    Nf = [2 * k * nx + 1, 2 * k * ny + 1, k * nzf + 1]
    nC = Nc[0] * Nc[1] * Nc[2]
    plane_c, plane_f = Nc[0] * Nc[1], Nf[0] * Nf[1]
    nF = plane_f * Nf[2]
    n = nC + nF - plane_f
    mc, mf = constrained_mask_fast(pc), constrained_mask_fast(pf)
    # fine interface plane = P2D (coarse top plane), coarse Dirichlet columns and fine
    # Dirichlet rows (the plane's boundary lines) dropped
    P2 = prolongation(k, (nx, ny), dim=2).tocoo()
    top = nC - plane_c
    keep = ~mc[top + P2.col] & ~mf[P2.row]
    rows = [P2.row[keep]]
    cols = [top + P2.col[keep]]
    vals = [P2.data[keep]]
    up = np.arange(plane_f, nF)
    rows.append(up)
    cols.append(nC + up - plane_f)
    vals.append(np.ones(up.size))
    E = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(nF, n))
    mask = np.concatenate([mc, mf[plane_f:]])
    return TwoBlock(pc, pf, E, nC, n, mask)


def _ext(A: sp.spmatrix, nC: int, n: int) -> sp.csr_matrix:
    A = A.tocoo()
    return sp.csr_matrix((A.data, (A.row, A.col)), shape=(n, n))


def _csr(p, which=0) -> sp.csr_matrix:
    C = CSR(p, which=which)
    return sp.csr_matrix((C.val, C.col, C.rowptr), shape=(C.n, C.n))


def operator(T: TwoBlock, which: int = 0) -> sp.csr_matrix:
    """A = A_c + E^T A_f E (which = 1: the mass matrix, same construction)."""
    Ac, Af = _csr(T.pc, which), _csr(T.pf, which)
    return (_ext(Ac, T.nc_dofs, T.n) + T.E.T @ Af @ T.E).tocsr()


def operator_unconstrained(T: TwoBlock, which: int = 0) -> sp.csr_matrix:
    """The same construction without the Dirichlet identity convention: every coarse
    interface node (boundary lines included) prolongated, unmodified block matrices."""
    k, nx, ny = T.pc.degree, T.pc.nc[0], T.pc.nc[1]
    plane_c = (k * nx + 1) * (k * ny + 1)
    plane_f = (2 * k * nx + 1) * (2 * k * ny + 1)
    nF = T.E.shape[0]
    P2 = prolongation(k, (nx, ny), dim=2).tocoo()
    top = T.nc_dofs - plane_c
    up = np.arange(plane_f, nF)
    E = sp.csr_matrix((np.concatenate([P2.data, np.ones(up.size)]),
                       (np.concatenate([P2.row, up]), np.concatenate([top + P2.col, T.nc_dofs + up - plane_f]))),
                      shape=(nF, T.n))
    Ac = CSR(T.pc, which=which, dirichlet=False)
    Af = CSR(T.pf, which=which, dirichlet=False)
    Ac = sp.csr_matrix((Ac.val, Ac.col, Ac.rowptr), shape=(Ac.n, Ac.n))
    Af = sp.csr_matrix((Af.val, Af.col, Af.rowptr), shape=(Af.n, Af.n))
    return (_ext(Ac, T.nc_dofs, T.n) + E.T @ Af @ E).tocsr()


def load(T: TwoBlock, f_kind: int = 1) -> np.ndarray:
    """b = b_c + E^T b_f (O8 right-hand sides of the two blocks, zero on Dirichlet DoFs)."""
    b = np.zeros(T.n)
    b[:T.nc_dofs] = rhs(T.pc, f_kind)
    return b + T.E.T @ rhs(T.pf, f_kind)


def error(T: TwoBlock, u: np.ndarray) -> float:
    """L2 error of the manufactured solution over both blocks (Gauss(k+3), R14)."""
    return float(np.hypot(l2_error(T.pc, u[:T.nc_dofs]), l2_error(T.pf, T.E @ u)))


def node_coords(T: TwoBlock) -> np.ndarray:
    """Physical coordinates of the global DoFs, [n, 3]."""
    out = []
    for p, skip in ((T.pc, 0), (T.pf, 1)):
        N = [p.degree * p.nc[e] + 1 for e in range(3)]
        axes = [np.linspace(p.lo[e], p.hi[e], p.nc[e] + 1) for e in range(3)]
        from . import gll

        xi = gll(p.degree)
        pts = []
        for e in range(3):
            h = (p.hi[e] - p.lo[e]) / p.nc[e]
            pts.append(np.array([p.lo[e] + h * (c + xi[j]) for c in range(p.nc[e]) for j in range(p.degree)]
                                + [p.hi[e]]))
        Z, Y, X = np.meshgrid(pts[2], pts[1], pts[0], indexing="ij")
        xyz = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
        out.append(xyz[skip * N[0] * N[1]:])
        del axes
    return np.concatenate(out)
