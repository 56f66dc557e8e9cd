"""Pins for the oracle's 1D rules and basis (O1, O2) against closed forms and
independent library routines (numpy.polynomial.legendre).  CPU only."""
import json
import os
from math import sqrt  # noqa: F401  (used by eval of the closed forms)

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _closed(s):
    return eval(s, {"sqrt": sqrt})


def test_gll_gauss_closed_forms():
    g = json.load(open(os.path.join(GOLDEN, "gll_gauss_closed_forms.json")))
    tol = g["tol"]
    for k, nodes in g["gll"].items():
        x = oracle.gll(int(k))
        np.testing.assert_allclose(x, [_closed(s) for s in nodes], rtol=0, atol=tol)
    for n, d in g["gauss"].items():
        x, w = oracle.gauss(int(n))
        np.testing.assert_allclose(x, [_closed(s) for s in d["x"]], rtol=0, atol=tol)
        np.testing.assert_allclose(w, [_closed(s) for s in d["w"]], rtol=0, atol=tol)


@pytest.mark.parametrize("k", range(1, 11))
def test_gll_are_roots_of_legendre_derivative(k):
    # independent: numpy's Legendre class, roots of P_k' on [-1,1]
    from numpy.polynomial import legendre as L

    ref = np.sort(np.concatenate([[-1.0, 1.0], L.Legendre.basis(k).deriv().roots()])) if k > 1 else np.array([-1.0, 1.0])
    np.testing.assert_allclose(oracle.gll(k), 0.5 * (1 + ref), rtol=0, atol=2e-15)


@pytest.mark.parametrize("n", range(1, 13))
def test_gauss_matches_leggauss_and_exactness(n):
    t, wt = np.polynomial.legendre.leggauss(n)
    x, w = oracle.gauss(n)
    np.testing.assert_allclose(x, 0.5 * (1 + t), rtol=0, atol=2e-15)
    np.testing.assert_allclose(w, 0.5 * wt, rtol=0, atol=2e-15)
    assert abs(w.sum() - 1.0) < 1e-15
    for m in range(2 * n):  # exact to degree 2n-1 (QGauss(3) integrates x^5)
        assert abs((w * x**m).sum() - 1.0 / (m + 1)) < 2e-15
    # not exact at degree 2n: error = (n!)^4 / ((2n+1) ((2n)!)^2) for x^(2n) on [0,1]
    from math import factorial as f

    err = f(n) ** 4 / ((2 * n + 1) * f(2 * n) ** 2)
    assert abs(1.0 / (2 * n + 1) - (w * x ** (2 * n)).sum() - err) < 1e-15 + 1e-9 * err


@pytest.mark.parametrize("k", range(1, 9))
def test_lagrange_kronecker_pou_fd(k):
    nodes = oracle.gll(k)
    n = k + 1
    for i in range(n):
        for j in range(n):
            assert abs(oracle.lagrange(nodes, i, nodes[j]) - (i == j)) < 1e-12
    rng = np.random.default_rng(k)
    for x in rng.random(20):
        assert abs(sum(oracle.lagrange(nodes, i, x) for i in range(n)) - 1.0) < 1e-13
        assert abs(sum(oracle.lagrange_d(nodes, i, x) for i in range(n))) < 1e-11
        for i in range(n):
            h = 1e-6
            fd = (oracle.lagrange(nodes, i, x + h) - oracle.lagrange(nodes, i, x - h)) / (2 * h)
            assert abs(fd - oracle.lagrange_d(nodes, i, x)) < 1e-6 * max(1, k * k)


@pytest.mark.parametrize("k", range(1, 9))
def test_lagrange_matches_polyfit(k):
    # independent: the interpolating polynomial through (nodes, e_i) by numpy Polynomial
    from numpy.polynomial import Polynomial

    nodes = oracle.gll(k)
    for i in range(k + 1):
        P = Polynomial.fit(nodes, np.eye(k + 1)[i], k, domain=[0, 1])  # window [-1,1]: well conditioned
        for x in np.linspace(0, 1, 7):
            assert abs(P(x) - oracle.lagrange(nodes, i, x)) < 1e-11
            assert abs(P.deriv()(x) - oracle.lagrange_d(nodes, i, x)) < 1e-9
