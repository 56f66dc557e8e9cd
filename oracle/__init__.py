"""CPU oracle for the matrix-free Laplace hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_1910_13247_b200`` (the CUDA path) and never
imports it.  The arithmetic lives in ``oracle.c`` (plain C + OpenMP, fp64);
this module is a ctypes binding plus the solver algorithms of SURVEY.md
§8(c) O9-O11 written out in numpy (``solvers.py``).

Parity status: every routine is pinned by a
``-m "not gpu"`` test against closed forms / exact integration / brute force.
The variable-coefficient operator on the deformed mesh has no closed form; it
is pinned by invariants (Neumann kernel, symmetry, linears) and by the energy
of the physical linears, u_a^T A u_b = delta_ab int c dx, against a mesh-free
quadrature of int c (tests/test_oracle_operator.py::
test_deformed_variable_coefficient_energy_of_linears).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2 -fopenmp)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-Wall",
             "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


class Problem(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("nc", ctypes.c_int64 * 3),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("degree", ctypes.c_int32),
        ("geom", ctypes.c_int32),
        ("eps", ctypes.c_double),
        ("coeff_kind", ctypes.c_int32),
        ("coeff_value", ctypes.c_double),
        ("dirichlet", ctypes.c_uint32),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER(Problem)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        sig = {
            "or_gauss": (ctypes.c_int, [ctypes.c_int, dp, dp]),
            "or_gll": (ctypes.c_int, [ctypes.c_int, dp]),
            "or_lagrange": (ctypes.c_double, [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double]),
            "or_lagrange_d": (ctypes.c_double, [dp, ctypes.c_int, ctypes.c_int, ctypes.c_double]),
            "or_n_dofs": (ctypes.c_int64, [P]),
            "or_n_cells": (ctypes.c_int64, [P]),
            "or_is_constrained": (ctypes.c_int, [P, ctypes.c_int64]),
            "or_cell_dofs": (ctypes.c_int, [P, ctypes.c_int64, i64p]),
            "or_phi": (None, [P, dp, dp]),
            "or_cell_matrix": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_int, dp, dp]),
            "or_csr_nnz": (ctypes.c_int64, [P]),
            "or_assemble_csr": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, i64p, i32p, dp]),
            "or_spmv": (None, [ctypes.c_int64, i64p, i32p, dp, dp, dp]),
            "or_csr_diagonal": (None, [ctypes.c_int64, i64p, i32p, dp, dp]),
            "or_apply_rows": (ctypes.c_int, [P, i64p, ctypes.c_int64, dp, dp]),
            "or_rhs": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, dp]),
            "or_l2_error": (ctypes.c_double, [P, dp, ctypes.c_int]),
            "or_kron_apply": (ctypes.c_int, [P, dp, dp]),
            "or_num_threads": (ctypes.c_int, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i64p(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _i32p(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def problem(dim=3, n_cells=(4, 4, 4), degree=2, lower=(0.0, 0.0, 0.0), upper=(1.0, 1.0, 1.0),
            geom=0, eps=0.1, coeff_kind=0, coeff_value=1.0, dirichlet=None) -> Problem:
    """Oracle problem descriptor.  dirichlet=None -> all 2*dim faces (R3)."""
    p = Problem()
    p.dim = dim
    nc = list(n_cells) + [1] * (3 - len(n_cells))
    for e in range(3):
        p.nc[e] = int(nc[e]) if e < dim else 1
        p.lo[e] = float(lower[e]) if e < len(lower) else 0.0
        p.hi[e] = float(upper[e]) if e < len(upper) else 1.0
    p.degree = degree
    p.geom = geom
    p.eps = eps
    p.coeff_kind = coeff_kind
    p.coeff_value = coeff_value
    p.dirichlet = ((1 << (2 * dim)) - 1) if dirichlet is None else int(dirichlet)
    return p


# --- 1D rules (O1, O2) -------------------------------------------------------
def gauss(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    lib().or_gauss(n, _dp(x), _dp(w))
    return x, w


def gll(k: int):
    x = np.zeros(k + 1)
    lib().or_gll(k, _dp(x))
    return x


def lagrange(nodes: np.ndarray, i: int, x: float) -> float:
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    return lib().or_lagrange(_dp(nodes), len(nodes), i, x)


def lagrange_d(nodes: np.ndarray, i: int, x: float) -> float:
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    return lib().or_lagrange_d(_dp(nodes), len(nodes), i, x)


# --- mesh / element (O3-O5) --------------------------------------------------
def n_dofs(p: Problem) -> int:
    return lib().or_n_dofs(ctypes.byref(p))


def constrained_mask(p: Problem) -> np.ndarray:
    n = n_dofs(p)
    L = lib()
    return np.array([L.or_is_constrained(ctypes.byref(p), g) for g in range(n)], dtype=bool)


def constrained_mask_fast(p: Problem) -> np.ndarray:
    """Same as constrained_mask, vectorised over the brick's 1D node grid."""
    N = [p.degree * p.nc[e] + 1 if e < p.dim else 1 for e in range(3)]
    m = np.zeros((N[2], N[1], N[0]), dtype=bool)
    ax = {0: 2, 1: 1, 2: 0}
    for e in range(p.dim):
        if (p.dirichlet >> (2 * e)) & 1:
            sl = [slice(None)] * 3
            sl[ax[e]] = 0
            m[tuple(sl)] = True
        if (p.dirichlet >> (2 * e + 1)) & 1:
            sl = [slice(None)] * 3
            sl[ax[e]] = N[e] - 1
            m[tuple(sl)] = True
    return m.reshape(-1)


def cell_dofs(p: Problem, cell: int) -> np.ndarray:
    nv = (p.degree + 1) ** p.dim
    d = np.zeros(nv, dtype=np.int64)
    lib().or_cell_dofs(ctypes.byref(p), cell, _i64p(d))
    return d


def cell_matrix(p: Problem, cell: int = 0, nq: int | None = None, mass: bool = False):
    nv = (p.degree + 1) ** p.dim
    A = np.zeros((nv, nv))
    M = np.zeros((nv, nv))
    st = lib().or_cell_matrix(ctypes.byref(p), cell, nq or p.degree + 1, _dp(A), _dp(M))
    if st != 0:
        raise FloatingPointError("det J <= 0 (SingularTensor)")
    return (A, M) if mass else A


class CSR:
    """Assembled global matrix (O6) with SpMV (O7)."""

    def __init__(self, p: Problem, which: int = 0, dirichlet: bool = True):
        L = lib()
        self.n = n_dofs(p)
        nnz = L.or_csr_nnz(ctypes.byref(p))
        self.rowptr = np.zeros(self.n + 1, dtype=np.int64)
        self.col = np.zeros(nnz, dtype=np.int32)
        self.val = np.zeros(nnz, dtype=np.float64)
        st = L.or_assemble_csr(ctypes.byref(p), which, 1 if dirichlet else 0,
                               _i64p(self.rowptr), _i32p(self.col), _dp(self.val))
        if st != 0:
            raise FloatingPointError("det J <= 0 (SingularTensor)")
        self.nnz = nnz

    def matvec(self, x: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n) if out is None else out
        lib().or_spmv(self.n, _i64p(self.rowptr), _i32p(self.col), _dp(self.val), _dp(x), _dp(y))
        return y

    __matmul__ = matvec

    def diagonal(self) -> np.ndarray:
        d = np.zeros(self.n)
        lib().or_csr_diagonal(self.n, _i64p(self.rowptr), _i32p(self.col), _dp(self.val), _dp(d))
        return d

    def dense(self) -> np.ndarray:
        D = np.zeros((self.n, self.n))
        for i in range(self.n):
            s, e = self.rowptr[i], self.rowptr[i + 1]
            D[i, self.col[s:e]] += self.val[s:e]
        return D


def apply_rows(p: Problem, rows: np.ndarray, x: np.ndarray) -> np.ndarray:
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(len(rows))
    st = lib().or_apply_rows(ctypes.byref(p), _i64p(rows), len(rows), _dp(x), _dp(out))
    if st != 0:
        raise FloatingPointError("det J <= 0 (SingularTensor)")
    return out


def rhs(p: Problem, f_kind: int = 0, nq: int | None = None) -> np.ndarray:
    b = np.zeros(n_dofs(p))
    lib().or_rhs(ctypes.byref(p), f_kind, nq or p.degree + 1, _dp(b))
    return b


def l2_error(p: Problem, u: np.ndarray, nq: int | None = None) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    return lib().or_l2_error(ctypes.byref(p), _dp(u), nq or p.degree + 3)


def kron_apply(p: Problem, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    if lib().or_kron_apply(ctypes.byref(p), _dp(x), _dp(y)) != 0:
        raise ValueError("Kronecker oracle needs an affine brick with constant coefficient")
    return y


def num_threads() -> int:
    return lib().or_num_threads()
