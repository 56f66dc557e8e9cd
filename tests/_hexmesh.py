"""Test-side builders of unstructured hex inputs.

`conforming(...)`: a (jittered, rotated, renumbered) brick from synth.hex_mesh, numbered
by the oracle's brute-force coordinate rule.  `two_block(...)`: the 2:1 hanging
interface of oracle/hanging.py (R20) written as an unstructured mesh with
constraint lines (R22): every fine interface node that is not a coarse node is the
coarse face function at that point, u = sum_ab l_a(xi) l_b(eta) u_ab over the coarse
top-face nodes, l the GLL Lagrange basis evaluated point by point here."""
from __future__ import annotations

import numpy as np

import oracle
import synth
from oracle import hex as ohex


def conforming(n_cells=(2, 2, 2), k=2, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0), jitter=0.2, seed=1,
               rotate=True, shuffle=True):
    V, C = synth.hex_mesh(n_cells, lower, upper, jitter=jitter, seed=seed, rotate=rotate, shuffle=shuffle)
    pts = ohex.support_points(V, C, k)
    cd, coords = ohex.number_by_coordinates(pts)
    return dict(vertices=V, cells=C, k=k, cell_dofs=cd, n_dofs=len(coords), coords=coords, lines=[],
                dirichlet=ohex.boundary_dofs(coords, lower, upper), lower=lower, upper=upper)


def two_block(n_cells=(2, 2, 1), nzf=2, k=2, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0), z_mid=0.5):
    nx, ny, nzc = n_cells
    Vc, Cc = synth.hex_mesh((nx, ny, nzc), lower, (upper[0], upper[1], z_mid), rotate=False, shuffle=False)
    Vf, Cf = synth.hex_mesh((2 * nx, 2 * ny, nzf), (lower[0], lower[1], z_mid), upper, rotate=False,
                            shuffle=False)
    V = np.concatenate([Vc, Vf])
    C = np.concatenate([Cc, Cf + len(Vc)]).astype(np.int32)
    pts = ohex.support_points(V, C, k)
    cd_all, coords_all = ohex.number_by_coordinates(pts)
    n_coarse_cells = len(Cc)
    coarse_dofs = np.unique(cd_all[:n_coarse_cells])
    on_iface = np.abs(coords_all[:, 2] - z_mid) < 1e-12
    hanging = np.nonzero(on_iface & ~np.isin(np.arange(len(coords_all)), coarse_dofs))[0]
    keep = np.setdiff1d(np.arange(len(coords_all)), hanging)
    new = -np.ones(len(coords_all), dtype=np.int64)
    new[keep] = np.arange(len(keep))
    coords = coords_all[keep]
    # constraint line of each hanging node: the coarse face interpolant
    nodes = oracle.gll(k)
    hc = (np.asarray(upper[:2]) - np.asarray(lower[:2])) / np.array([nx, ny])
    key = {tuple(np.round(p / 1e-9).astype(np.int64)): d for d, p in enumerate(coords)}
    lines = []
    line_of = {}
    for hd in hanging:
        x, y = coords_all[hd, 0], coords_all[hd, 1]
        cx = min(int((x - lower[0]) // hc[0]), nx - 1)
        cy = min(int((y - lower[1]) // hc[1]), ny - 1)
        x0, y0 = lower[0] + cx * hc[0], lower[1] + cy * hc[1]
        xi, eta = (x - x0) / hc[0], (y - y0) / hc[1]
        line = []
        for b in range(k + 1):
            for a in range(k + 1):
                w = oracle.lagrange(nodes, a, xi) * oracle.lagrange(nodes, b, eta)
                if abs(w) < 1e-15:
                    continue
                p = np.array([x0 + nodes[a] * hc[0], y0 + nodes[b] * hc[1], z_mid])
                line.append((key[tuple(np.round(p / 1e-9).astype(np.int64))], w))
        line_of[hd] = len(lines)
        lines.append(line)
    cd = np.empty_like(cd_all)
    for c in range(len(C)):
        for i in range(cd_all.shape[1]):
            d = cd_all[c, i]
            cd[c, i] = new[d] if new[d] >= 0 else -1 - line_of[d]
    return dict(vertices=V, cells=C, k=k, cell_dofs=cd, n_dofs=len(coords), coords=coords, lines=lines,
                dirichlet=ohex.boundary_dofs(coords, lower, upper), lower=lower, upper=upper)


def oracle_matrix(m, coeff="constant", value=1.0, dirichlet=True, mass=False):
    return ohex.assemble(m["vertices"], m["cells"], m["k"], m["cell_dofs"], m["n_dofs"], m["lines"],
                         m["dirichlet"] if dirichlet else None, coeff, value, mass=mass)


def match(coords_a: np.ndarray, coords_b: np.ndarray) -> np.ndarray:
    """perm with coords_b[perm[j]] == coords_a[j] (within 1e-9)."""
    key = {tuple(np.round(p / 1e-9).astype(np.int64)): i for i, p in enumerate(coords_b)}
    return np.array([key[tuple(np.round(p / 1e-9).astype(np.int64))] for p in coords_a], dtype=np.int64)
