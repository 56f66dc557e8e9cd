"""DG-SIP oracle -- TEST INFRASTRUCTURE ONLY.

The symmetric interior penalty discontinuous Galerkin Laplacian that the paper's
§6.1 experiment times ("a symmetric interior penalty
discontinuous Galerkin discretization with polynomial degree p = 4 on a
hyper-rectangle"), written out as its plain definition on a brick of n_x x n_y x
n_z axis-aligned cells:

  a(u, v) = sum_K (grad u, grad v)_K
          + sum_{interior F} ( -({d_n u}, [v])_F - ([u], {d_n v})_F + sigma_F ([u], [v])_F )
          + sum_{boundary F} ( -(d_n u, v)_F - (u, d_n v)_F + sigma_F (u, v)_F )

[w] = w^- - w^+ and {w} = (w^- + w^+)/2 across F with n pointing from K^- (lower
coordinate) to K^+; on boundary faces n is the outward normal (weak, Nitsche-type
homogeneous Dirichlet on every face).  Readings (R16-R18): discontinuous
Q_k Lagrange basis on the GLL nodes of each cell (DoF index = cell (k+1)^3 + local,
both x-fastest); Gauss(k+1) quadrature on cells and faces; penalty
sigma_F = 2 (k+1)^2 / h_n, h_n the cell size normal to F.

Cell matrices come from the CG oracle's brute-force cell integral (oracle.c,
pinned); face integrals are evaluated here point by point from the oracle's
Lagrange product formula.  Pins: tests/test_oracle_dg.py.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import cell_matrix, gauss, gll, lagrange, lagrange_d, problem


def penalty(k: int, h_n: float) -> float:
    """R17: sigma_F = 2 (k+1)^2 / h_n."""
    return 2.0 * (k + 1) ** 2 / h_n


def _cells(n_cells):
    nx, ny, nz = n_cells
    return nx * ny * nz


def _cell_index(c, n_cells):
    return c[0] + n_cells[0] * (c[1] + n_cells[1] * c[2])


def n_dofs(n_cells, k):
    return _cells(n_cells) * (k + 1) ** 3


def _face_traces(k, axis, side, h, xq):
    """Values and normal (x_axis) derivatives of the N^3 cell basis functions at the
    face quadrature points of the cell face xi_axis = side (0 or 1).
    Returns V[q, i], Dn[q, i] with q over the (k+1)^2 tangential Gauss points."""
    nodes = gll(k)
    N = k + 1
    t1, t2 = [a for a in range(3) if a != axis]
    V = np.zeros((N * N, N ** 3))
    D = np.zeros((N * N, N ** 3))
    for qa in range(N):
        for qb in range(N):
            q = qa + N * qb
            for i in range(N ** 3):
                idx = (i % N, (i // N) % N, i // (N * N))
                tang = lagrange(nodes, idx[t1], xq[qa]) * lagrange(nodes, idx[t2], xq[qb])
                V[q, i] = lagrange(nodes, idx[axis], float(side)) * tang
                D[q, i] = lagrange_d(nodes, idx[axis], float(side)) / h[axis] * tang
    return V, D


def assemble(n_cells, k, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0)) -> sp.csr_matrix:
    n_cells = tuple(int(c) for c in n_cells)
    N = k + 1
    nb = N ** 3
    h = [(upper[e] - lower[e]) / n_cells[e] for e in range(3)]
    p = problem(dim=3, n_cells=n_cells, degree=k, lower=lower, upper=upper, dirichlet=0)
    rows, cols, vals = [], [], []

    def add(bi, bj, block):
        r = np.repeat(np.arange(nb) + bi * nb, nb)
        c = np.tile(np.arange(nb) + bj * nb, nb)
        rows.append(r)
        cols.append(c)
        vals.append(block.ravel())

    # cell terms (the same cell integral as the CG operator)
    for cell in range(_cells(n_cells)):
        add(cell, cell, cell_matrix(p, cell))
    # face terms
    xq, wq = gauss(N)
    for axis in range(3):
        t1, t2 = [a for a in range(3) if a != axis]
        wf = np.outer(wq, wq).T.ravel() * h[t1] * h[t2]  # weight of q = qa + N qb
        sig = penalty(k, h[axis])
        Vm, Dm = _face_traces(k, axis, 1, h, xq)  # K^- side (its xi_axis = 1)
        Vp, Dp = _face_traces(k, axis, 0, h, xq)  # K^+ side (its xi_axis = 0)
        # interior face blocks: B[s_i][s_j] = sum_q w ( -{dn phi_j}[phi_i] - [phi_j]{dn phi_i} + sig [phi_j][phi_i] )
        J = {"-": Vm, "+": -Vp}          # [phi] per side
        Avg = {"-": 0.5 * Dm, "+": 0.5 * Dp}  # {d_n phi} per side (n = +e_axis)
        blocks = {}
        for si in "-+":
            for sj in "-+":
                blocks[si, sj] = (-(J[si] * wf[:, None]).T @ Avg[sj] - (Avg[si] * wf[:, None]).T @ J[sj]
                                  + sig * (J[si] * wf[:, None]).T @ J[sj])
        # boundary faces: low end (outward n = -e, cell side xi = 0) and high end (n = +e, xi = 1)
        bl = -(Vp * wf[:, None]).T @ (-Dp) - ((-Dp) * wf[:, None]).T @ Vp + sig * (Vp * wf[:, None]).T @ Vp
        bh = -(Vm * wf[:, None]).T @ Dm - (Dm * wf[:, None]).T @ Vm + sig * (Vm * wf[:, None]).T @ Vm
        for cz in range(n_cells[2]):
            for cy in range(n_cells[1]):
                for cx in range(n_cells[0]):
                    c = [cx, cy, cz]
                    K = _cell_index(c, n_cells)
                    if c[axis] == 0:
                        add(K, K, bl)
                    if c[axis] == n_cells[axis] - 1:
                        add(K, K, bh)
                    else:
                        c2 = list(c)
                        c2[axis] += 1
                        Kp = _cell_index(c2, n_cells)
                        add(K, K, blocks["-", "-"])
                        add(K, Kp, blocks["-", "+"])
                        add(Kp, K, blocks["+", "-"])
                        add(Kp, Kp, blocks["+", "+"])
    n = n_dofs(n_cells, k)
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


def node_coords(n_cells, k, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0)) -> np.ndarray:
    """Physical coordinates of every DG DoF, [n, 3]."""
    N = k + 1
    nodes = gll(k)
    h = [(upper[e] - lower[e]) / n_cells[e] for e in range(3)]
    X = np.zeros((n_dofs(n_cells, k), 3))
    g = 0
    for cz in range(n_cells[2]):
        for cy in range(n_cells[1]):
            for cx in range(n_cells[0]):
                for i in range(N ** 3):
                    idx = (i % N, (i // N) % N, i // (N * N))
                    c = (cx, cy, cz)
                    X[g] = [lower[e] + h[e] * (c[e] + nodes[idx[e]]) for e in range(3)]
                    g += 1
    return X


def rhs(n_cells, k, f, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0)) -> np.ndarray:
    """b_i = sum_K int_K f phi_i with Gauss(k+1) (homogeneous weak Dirichlet: no face terms)."""
    N = k + 1
    nodes = gll(k)
    xq, wq = gauss(N)
    h = [(upper[e] - lower[e]) / n_cells[e] for e in range(3)]
    L = np.array([[lagrange(nodes, i, x) for x in xq] for i in range(N)])  # [i, q]
    b = np.zeros(n_dofs(n_cells, k))
    g = 0
    for cz in range(n_cells[2]):
        for cy in range(n_cells[1]):
            for cx in range(n_cells[0]):
                c = (cx, cy, cz)
                X = [lower[e] + h[e] * (c[e] + xq) for e in range(3)]
                F = f(X[0][:, None, None], X[1][None, :, None], X[2][None, None, :])  # [qx, qy, qz]
                W = np.einsum("a,b,c->abc", wq, wq, wq) * h[0] * h[1] * h[2]
                bc = np.einsum("ia,jb,kc,abc->kji", L, L, L, F * W)  # [k, j, i] -> x fastest
                b[g:g + N ** 3] = bc.ravel()
                g += N ** 3
    return b


def l2_error(n_cells, k, u, exact, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0)) -> float:
    """(sum_K int_K (u_h - u)^2)^(1/2) with Gauss(k+3) (R14)."""
    N = k + 1
    nodes = gll(k)
    xq, wq = gauss(k + 3)
    h = [(upper[e] - lower[e]) / n_cells[e] for e in range(3)]
    L = np.array([[lagrange(nodes, i, x) for x in xq] for i in range(N)])
    err = 0.0
    g = 0
    for cz in range(n_cells[2]):
        for cy in range(n_cells[1]):
            for cx in range(n_cells[0]):
                c = (cx, cy, cz)
                X = [lower[e] + h[e] * (c[e] + xq) for e in range(3)]
                uc = u[g:g + N ** 3].reshape(N, N, N)  # [k, j, i]
                uh = np.einsum("kji,ia,jb,kc->abc", uc, L, L, L)
                ex = exact(X[0][:, None, None], X[1][None, :, None], X[2][None, None, :])
                W = np.einsum("a,b,c->abc", wq, wq, wq) * h[0] * h[1] * h[2]
                err += float(np.sum((uh - ex) ** 2 * W))
                g += N ** 3
    return err ** 0.5
