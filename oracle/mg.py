"""Geometric multigrid oracle -- TEST INFRASTRUCTURE ONLY.

Plain numpy / scipy.sparse definitions, written from the paper and the SPEC's
multigrid module:

* hierarchy: a globally refined brick, level l has n_cells(L) / 2^(L-l) cells per
  direction, the same degree k on every level (§6.1: "progresses
  to coarser mesh levels until a coarse solver is invoked");
* prolongation = interpolation of the coarse finite-element function at the fine
  support points ("space embedding"); on the tensor-product brick it is
  P = Pz (x) Py (x) Px with the 1D matrix P1[f, c] = phi_c(x_f), evaluated here with
  the oracle's own Lagrange product formula; restriction R = P^T;
  homogeneous Dirichlet: constrained fine rows and coarse columns are dropped
  (the identity-row convention R3 keeps constrained entries of every level at 0);
* smoother: the Chebyshev(6) polynomial of solvers.chebyshev on [lam_l/20, lam_l],
  lam_l = 1.2 Ritz(12) of the level operator ("Chebyshev smoothing of degree 6
  for pre- and post-smoothing"): pre-smoothing from x = 0,
  post-smoothing x += Cheb(b - A x);
* coarse solver: a dense direct solve ("dense factorization");
* V-cycle: pre-smooth, residual, restrict, recurse, prolongate and
  correct, post-smooth.

Pins: tests/test_oracle_mg.py (polynomial reproduction of the prolongation in 1D
and 3D, partition of unity, the Q1 midpoint rule, the Galerkin identity
R A_f P = A_c on affine meshes, linearity / symmetry of the V-cycle, mesh-
independent convergence rates, MG-PCG iteration counts).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

import synth

from . import CSR, constrained_mask_fast, gll, lagrange, n_dofs, problem
from .solvers import chebyshev, pcg, ritz_lambda_max


def prolongation_1d(k: int, n_coarse: int) -> np.ndarray:
    """P1[f, c] = phi_c(x_f): coarse Q_k basis (GLL nodes) at the fine 1D nodes.
    Coordinates in coarse-cell units: coarse cell cc = [cc, cc + 1]; fine node
    f = k fc + m sits at (fc + xi_m) / 2."""
    xi = gll(k)
    nf, nc = 2 * k * n_coarse + 1, k * n_coarse + 1
    P = np.zeros((nf, nc))
    for f in range(nf):
        fc, m = divmod(f, k)
        if fc == 2 * n_coarse:  # the last node
            fc, m = fc - 1, k
        x = 0.5 * (fc + xi[m])
        cc = min(int(np.floor(x)), n_coarse - 1)
        t = x - cc
        for j in range(k + 1):
            P[f, k * cc + j] = lagrange(xi, j, t)
    return P


def prolongation(k: int, n_coarse_cells, dim: int = 3) -> sp.csr_matrix:
    """P = Pz (x) Py (x) Px (lexicographic, x fastest)."""
    mats = [sp.csr_matrix(prolongation_1d(k, int(n_coarse_cells[e]))) for e in range(dim)]
    P = mats[0]
    for e in range(1, dim):
        P = sp.kron(mats[e], P, format="csr")
    return P


@dataclass
class Level:
    p: object
    A: CSR
    diag: np.ndarray
    lam: float
    mask: np.ndarray  # constrained DoFs


@dataclass
class Hierarchy:
    levels: list = field(default_factory=list)
    P: list = field(default_factory=list)  # P[l] maps level l-1 -> l (masked)
    coarse_dense: np.ndarray | None = None
    degree: int = 6
    smoothing_range: float = 20.0


def n_levels_auto(n_cells, max_coarse_dofs: int, k: int, dim: int = 3) -> int:
    """Levels by halving while every direction is even and the coarser level still has
    more than max_coarse_dofs DoFs (the coarse level is the first one at or below it)."""
    nc = list(n_cells[:dim])
    L = 1
    while all(c % 2 == 0 for c in nc) and np.prod([k * c + 1 for c in nc]) > max_coarse_dofs:
        nc = [c // 2 for c in nc]
        L += 1
    return L


def build_hierarchy(dim=3, n_cells=(8, 8, 8), k=2, n_levels=None, max_coarse_dofs=1000, safety=1.2,
                    eig_steps=12, degree=6, smoothing_range=20.0, **problem_kw) -> Hierarchy:
    n_cells = tuple(n_cells[:dim])
    if n_levels is None:
        n_levels = n_levels_auto(n_cells, max_coarse_dofs, k, dim)
    H = Hierarchy(degree=degree, smoothing_range=smoothing_range)
    for l in range(n_levels):
        f = 2 ** (n_levels - 1 - l)
        if any(c % f for c in n_cells):
            raise ValueError("n_cells not divisible by 2^(levels-1)")
        ncl = tuple(c // f for c in n_cells)
        p = problem(dim=dim, n_cells=ncl, degree=k, **problem_kw)
        A = CSR(p)
        d = A.diagonal()
        mask = constrained_mask_fast(p)
        s = synth.with_zero_dirichlet(synth.vector(A.n, 0), mask)
        lam = safety * ritz_lambda_max(A.matvec, d, s, eig_steps)
        H.levels.append(Level(p, A, d, lam, mask))
        if l > 0:
            prev = H.levels[l - 1]
            P = prolongation(k, [prev.p.nc[e] for e in range(dim)], dim)
            Df = sp.diags((~mask).astype(float))
            Dc = sp.diags((~prev.mask).astype(float))
            H.P.append((Df @ P @ Dc).tocsr())
        else:
            H.P.append(None)
    H.coarse_dense = H.levels[0].A.dense()
    return H


def prolongate(H: Hierarchy, l: int, xc: np.ndarray) -> np.ndarray:
    return H.P[l] @ xc


def restrict(H: Hierarchy, l: int, rf: np.ndarray) -> np.ndarray:
    return H.P[l].T @ rf


def smooth(H: Hierarchy, l: int, b: np.ndarray, x: np.ndarray | None = None) -> np.ndarray:
    L = H.levels[l]
    if x is None:
        return chebyshev(L.A.matvec, L.diag, b, L.lam, H.degree, H.smoothing_range)
    return x + chebyshev(L.A.matvec, L.diag, b - L.A @ x, L.lam, H.degree, H.smoothing_range)


def vcycle(H: Hierarchy, b: np.ndarray, l: int | None = None) -> np.ndarray:
    """pre-smooth, residual, restrict, recurse (dense solve on level 0),
    prolongate and correct, post-smooth."""
    if l is None:
        l = len(H.levels) - 1
    if l == 0:
        return np.linalg.solve(H.coarse_dense, b)
    L = H.levels[l]
    x = smooth(H, l, b)
    r = b - L.A @ x
    xc = vcycle(H, restrict(H, l, r), l - 1)
    x = x + prolongate(H, l, xc)
    return smooth(H, l, b, x)


def vcycle_rate(H: Hierarchy, b: np.ndarray, cycles: int = 10) -> float:
    """Geometric-mean residual reduction of the stationary iteration x += V(b - A x)."""
    A = H.levels[-1].A
    x = np.zeros_like(b)
    r0 = np.linalg.norm(b)
    r = b.copy()
    for _ in range(cycles):
        x = x + vcycle(H, r)
        r = b - A @ x
    return (np.linalg.norm(r) / r0) ** (1.0 / cycles)


def mg_pcg(H: Hierarchy, b: np.ndarray, rel_tol: float = 1e-10, max_iter: int = 1000):
    """CG on the finest level with one V-cycle as preconditioner."""
    A = H.levels[-1].A
    return pcg(A.matvec, b, lambda r: vcycle(H, r), rel_tol, max_iter)


__all__ = ["prolongation_1d", "prolongation", "build_hierarchy", "prolongate", "restrict", "smooth",
           "vcycle", "vcycle_rate", "mg_pcg", "n_levels_auto", "Hierarchy", "Level", "n_dofs"]
