"""Shared test helpers: build the oracle problem and the CUDA Operator from
one description, and compare element by element (R11)."""
from __future__ import annotations

import numpy as np

import oracle
import synth

CUDA_ORACLE_TOL = 1e-12  # north star: relative L2 agreement with the assembled oracle (R11)


def oracle_problem(case: dict):
    dim = case["dim"]
    return oracle.problem(
        dim=dim, n_cells=case["n_cells"], degree=case["k"], lower=case.get("lower", (0.0,) * 3),
        upper=case.get("upper", (1.0,) * 3), geom=1 if case.get("geometry") == "sine" else 0,
        eps=case.get("eps", 0.1), coeff_kind=1 if case.get("coeff") == "variable" else 0,
        coeff_value=case.get("coeff", 1.0) if case.get("coeff") != "variable" else 1.0,
        dirichlet=case.get("dirichlet"))


def cuda_operator(case: dict, **kw):
    from paper_1910_13247_b200 import Operator

    dim = case["dim"]
    return Operator(case["n_cells"], case["k"], dim=dim, lower=case.get("lower"), upper=case.get("upper"),
                    geometry=case.get("geometry", "cartesian"), eps=case.get("eps", 0.1),
                    coeff=case.get("coeff", 1.0), dirichlet_faces=case.get("dirichlet"), **kw)


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def seeded(n: int, seed: int) -> np.ndarray:
    return synth.vector(n, seed)
