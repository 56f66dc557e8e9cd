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
