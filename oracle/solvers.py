"""Oracle solvers -- TEST INFRASTRUCTURE ONLY.

Plain numpy transcriptions of the algorithms, in the order and notation of
DESIGN.md "Readings" R6-R9, R15 (from S:500-508 cg_solve, S:639-647
estimate_eigenvalue, S:648-656 chebyshev_apply, "Chebyshev smoothing
of degree 6").  ``A`` is any callable x -> A x (the CSR SpMV of the oracle).
Never imported by the product path.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class BreakdownError(RuntimeError):
    """p.Ap <= 0 or r.z <= 0."""


class MaxIterationsError(RuntimeError):
    """No convergence within max_iter."""


@dataclass
class CGResult:
    x: np.ndarray
    iterations: int
    final_rel_residual: float
    history: list = field(default_factory=list)  # ||r_j|| after each apply


def pcg(A, b: np.ndarray, precond, rel_tol: float = 1e-10, max_iter: int = 10000) -> CGResult:
    """O9: preconditioned CG from x0 = 0; stops when ||r||_2 <= tol ||b||_2 on
    the recursive residual; iterations = number of applications of A (R9)."""
    x = np.zeros_like(b)
    r = b.copy()
    normb = float(np.linalg.norm(b))
    if normb == 0.0:
        return CGResult(x, 0, 0.0, [])
    z = precond(r)
    p = z.copy()
    rz = float(r @ z)
    hist = []
    it = 0
    while True:
        v = A(p)
        it += 1
        pv = float(p @ v)
        if pv <= 0.0:
            raise BreakdownError("p.Ap <= 0")
        alpha = rz / pv
        x += alpha * p
        r -= alpha * v
        res = float(np.linalg.norm(r))
        hist.append(res)
        if res <= rel_tol * normb:
            return CGResult(x, it, res / normb, hist)
        if it >= max_iter:
            raise MaxIterationsError(f"{it} iterations, rel residual {res / normb:.3e}")
        z = precond(r)
        rz_new = float(r @ z)
        if rz_new <= 0.0:
            raise BreakdownError("r.z <= 0")
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new


def ritz_lambda_max(A, diag: np.ndarray, s: np.ndarray, n_steps: int = 12) -> float:
    """O10: largest Ritz value of D^{-1}A from n_steps Jacobi-PCG steps on
    A y = s (x0 = 0), tridiagonal T_jj = 1/a_j + b_{j-1}/a_{j-1},
    T_{j,j+1} = sqrt(b_j)/a_j (the CG-Lanczos relation).  Steps stop early
    when r.z falls below 1e-28 of its initial value (tiny problems converge
    exactly; R8)."""
    r = s.copy()
    z = r / diag
    p = z.copy()
    rz0 = rz = float(r @ z)
    alphas, betas = [], []
    for _ in range(n_steps):
        v = A(p)
        pv = float(p @ v)
        if pv <= 0.0:
            raise BreakdownError("p.Ap <= 0 in eigenvalue estimate")
        alpha = rz / pv
        alphas.append(alpha)
        r = r - alpha * v
        z = r / diag
        rz_new = float(r @ z)
        if rz_new <= 1e-28 * rz0:
            break
        beta = rz_new / rz
        betas.append(beta)
        p = z + beta * p
        rz = rz_new
    m = len(alphas)
    T = np.zeros((m, m))
    for j in range(m):
        T[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j > 0 else 0.0)
        if j + 1 < m:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(betas[j]) / alphas[j]
    return float(np.linalg.eigvalsh(T)[-1])


def chebyshev(A, diag: np.ndarray, r: np.ndarray, lam: float, degree: int = 6,
              smoothing_range: float = 20.0) -> np.ndarray:
    """O11: Chebyshev(degree) for D^{-1}A on [lam/range, lam] from x = 0 (R6, R7):
    x = D^{-1} r / theta; d = x; rho = 1/sigma;
    for j = 1..degree-1: rho' = 1/(2 sigma - rho);
        d = rho' rho d + (2 rho'/delta) D^{-1}(r - A x); x += d; rho = rho'."""
    a = lam / smoothing_range
    b = lam
    theta = 0.5 * (a + b)
    delta = 0.5 * (b - a)
    sigma = theta / delta
    x = r / diag / theta
    d = x.copy()
    rho = 1.0 / sigma
    for _ in range(degree - 1):
        rho_n = 1.0 / (2.0 * sigma - rho)
        d = rho_n * rho * d + (2.0 * rho_n / delta) * ((r - A(x)) / diag)
        x = x + d
        rho = rho_n
    return x


@dataclass
class ChebCGResult(CGResult):
    lambda_max: float = 0.0


def chebyshev_pcg(A, diag: np.ndarray, b: np.ndarray, s: np.ndarray, rel_tol: float = 1e-10,
                  max_iter: int = 10000, degree: int = 6, smoothing_range: float = 20.0,
                  safety: float = 1.2, eig_steps: int = 12) -> ChebCGResult:
    """The whole solver of §8(a) a10: lambda = safety * Ritz(eig_steps), then
    PCG preconditioned by Chebyshev(degree) on [lambda/range, lambda]."""
    lam = safety * ritz_lambda_max(A, diag, s, eig_steps)
    res = pcg(A, b, lambda r: chebyshev(A, diag, r, lam, degree, smoothing_range), rel_tol, max_iter)
    return ChebCGResult(res.x, res.iterations, res.final_rel_residual, res.history, lam)
