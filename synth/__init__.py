"""Seeded synthetic inputs shared by the oracle tests and the CUDA-path tests.

This module holds NONE of the method's arithmetic: it only draws numbers.
The generator is splitmix64 of a 64-bit counter (SURVEY.md §8(d) "Synthetic
inputs"; R8):

    z = counter + 0x9E3779B97F4A7C15
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB
    z =  z ^ (z >> 31)
    u = (z >> 11) * 2^-53  in [0,1);   value = 2u - 1  in [-1,1)

with counter = global DoF index + 2^40 * seed, so values are independent of
how the vector is partitioned.  The CUDA library implements the same counter
generator itself for the eigenvalue-estimate start vector (seed 0).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(counter: np.ndarray) -> np.ndarray:
    z = counter.astype(np.uint64) + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform(first: int, count: int, seed: int = 0) -> np.ndarray:
    """values for global indices [first, first+count) in [-1, 1), fp64."""
    with np.errstate(over="ignore"):
        c = np.arange(first, first + count, dtype=np.uint64) + np.uint64(seed) * np.uint64(1 << 40)
        z = splitmix64(c)
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def vector(n: int, seed: int = 0) -> np.ndarray:
    return uniform(0, n, seed)


def with_zero_dirichlet(v: np.ndarray, mask: np.ndarray) -> np.ndarray:
    out = v.copy()
    out[mask] = 0.0
    return out


# --- unstructured hexahedral meshes ----------------------
def _cube_rotations() -> list:
    """The 24 proper rotations of the cube as signed 3x3 permutation matrices."""
    import itertools

    out = []
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((1, -1), repeat=3):
            R = np.zeros((3, 3), dtype=np.int64)
            for r in range(3):
                R[r, perm[r]] = signs[r]
            if round(np.linalg.det(R)) == 1:
                out.append(R)
    return out


def hex_mesh(n_cells=(4, 4, 4), lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0), jitter: float = 0.0,
             seed: int = 0, rotate: bool = True, shuffle: bool = True):
    """A brick of nx x ny x nz hexahedra given as an unstructured mesh.

    Returns (vertices [nv][3] fp64, cell_vertices [nc][8] int32); a cell's vertices are
    listed lexicographically in its own local frame (local vertex a + 2 b + 4 c at
    reference corner (a, b, c)).  Interior vertices move by jitter * h * uniform[-1, 1)
    per axis (seeded); boundary vertices stay on the box faces.  With `rotate` every
    cell's local frame is one of the 24 proper cube rotations (drawn per cell), with
    `shuffle` the global vertex numbers are a seeded permutation -- neighbouring cells
    then disagree on edge / face orientation, as in a general hex mesh."""
    nx, ny, nz = n_cells
    nv = (nx + 1) * (ny + 1) * (nz + 1)
    ii, jj, ll = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    ijk = np.stack([ii.T.reshape(-1), jj.T.reshape(-1), ll.T.reshape(-1)], axis=1)  # x-fastest
    lo, hi = np.asarray(lower, dtype=np.float64), np.asarray(upper, dtype=np.float64)
    h = (hi - lo) / np.asarray(n_cells, dtype=np.float64)
    X = lo + ijk * h
    if jitter > 0.0:
        interior = np.all((ijk > 0) & (ijk < np.asarray(n_cells)), axis=1)
        d = uniform(0, 3 * nv, seed + 101).reshape(nv, 3)
        X[interior] += jitter * h * d[interior]
    perm = np.arange(nv)
    if shuffle:
        perm = np.argsort(uniform(0, nv, seed + 202), kind="stable")  # new id of old vertex v: inv
    new_id = np.empty(nv, dtype=np.int64)
    new_id[perm] = np.arange(nv)
    vertices = np.empty_like(X)
    vertices[new_id] = X
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cx, cy, cz = cx.reshape(-1), cy.reshape(-1), cz.reshape(-1)
    cells = np.empty((nx * ny * nz, 8), dtype=np.int64)
    for v in range(8):
        a, b, c = v & 1, (v >> 1) & 1, v >> 2
        cells[:, v] = new_id[((cz + c) * (ny + 1) + (cy + b)) * (nx + 1) + (cx + a)]
    if rotate:
        rots = _cube_rotations()
        pick = (np.abs(uniform(0, len(cells), seed + 303)) * len(rots)).astype(np.int64) % len(rots)
        out = np.empty_like(cells)
        corners = np.array([[v & 1, (v >> 1) & 1, v >> 2] for v in range(8)])
        for r, R in enumerate(rots):
            sel = pick == r
            if not sel.any():
                continue
            s = 2 * corners - 1
            t = (s @ R.T + 1) // 2  # corner v moves to local position t[v]
            dest = t[:, 0] + 2 * t[:, 1] + 4 * t[:, 2]
            out[np.ix_(sel, dest)] = cells[sel]
        cells = out
    return vertices, cells.astype(np.int32)
