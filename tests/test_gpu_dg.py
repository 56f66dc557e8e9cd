"""GPU parity of the DG-SIP operator against oracle/dg.py: the
apply element by element (relative L2 <= 1e-12, R11), the diagonal, and the
Chebyshev(6)-Jacobi PCG iteration counts (margin-guarded, R15)."""
import numpy as np
import pytest

import synth
from oracle import dg, solvers
from tests._helpers import rel_l2, seeded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


CASES = [
    dict(n_cells=(3, 2, 2), k=1),
    dict(n_cells=(2, 3, 2), k=2, upper=(1.0, 0.5, 2.0)),
    dict(n_cells=(3, 3, 3), k=3, coeff=2.5),
    dict(n_cells=(2, 2, 1), k=4),
    dict(n_cells=(1, 1, 1), k=5),
    dict(n_cells=(2, 1, 2), k=6),
    dict(n_cells=(2, 2, 1), k=7),
    dict(n_cells=(1, 2, 1), k=8),
    dict(n_cells=(5, 4, 3), k=2, upper=(2.0, 1.0, 0.5)),   # interior cells in every direction, ragged block
    dict(n_cells=(4, 3, 5), k=4),
]


def _op(c):
    from paper_1910_13247_b200 import Operator

    return Operator(c["n_cells"], c["k"], upper=c.get("upper"), coeff=c.get("coeff", 1.0), discretization="dg")


def _ref(c):
    return c.get("coeff", 1.0) * dg.assemble(c["n_cells"], c["k"], upper=c.get("upper", (1.0, 1.0, 1.0)))


def _id(c):
    return f"k{c['k']}-{'x'.join(map(str, c['n_cells']))}"


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_dg_apply_and_diagonal_match_oracle(case, torch):
    A = _ref(case)
    op = _op(case)
    assert op.n_local == A.shape[0]
    assert op.info()["apply_variant"] == 4
    for s in (1, 2, 3):
        x = seeded(A.shape[0], s)
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, A @ x) <= 1e-12, (s, rel_l2(y, A @ x))
    d = op.diagonal().cpu().numpy()
    assert np.abs(d - A.diagonal()).max() <= 1e-12 * np.abs(A.diagonal()).max()


@pytest.mark.parametrize("case", [CASES[1], CASES[2], dict(n_cells=(4, 4, 4), k=2)], ids=_id)
def test_dg_chebyshev_pcg_matches_oracle(case, torch):
    A = _ref(case)
    n = A.shape[0]
    d = A.diagonal()
    b = seeded(n, 11)
    s = synth.vector(n, 0)
    ref = solvers.chebyshev_pcg(lambda v: A @ v, d, b, s, rel_tol=1e-10)
    x, res = _op(case).cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-10)
    assert abs(res.lambda_max - ref.lambda_max) <= 1e-9 * ref.lambda_max
    normb = np.linalg.norm(b)
    h = ref.history
    if len(h) < 2 or min(h[-2] / (1e-10 * normb) - 1.0, 1.0 - h[-1] / (1e-10 * normb)) > 1e-6:
        assert res.iterations == ref.iterations
    assert rel_l2(x.cpu().numpy(), ref.x) <= 1e-8


def test_full_size_dg4_sampled_cells(torch):
    """bench.py's dg4 operator (Q4, 64^3 cells, 32.8 M DoFs) on a seeded vector, in the launch
    configuration bench.py times; sampled cells (corners, faces, interior) checked against the
    oracle on the clipped 3x3x3 sub-brick around each: a cell's rows involve only its six
    neighbours, the local h and, on domain faces, the Nitsche terms, all of which the
    sub-brick reproduces exactly."""
    from paper_1910_13247_b200 import Operator

    n, k = 64, 4
    NV = (k + 1) ** 3
    op = Operator((n, n, n), k, discretization="dg")
    x = seeded(op.n_local, 5)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    h = 1.0 / n
    for cell in [(0, 0, 0), (63, 63, 63), (31, 17, 45), (0, 40, 12), (63, 5, 0), (20, 63, 33), (1, 1, 62)]:
        lo = [max(0, c - 1) for c in cell]
        hi = [min(n - 1, c + 1) for c in cell]
        ns = [b - a + 1 for a, b in zip(lo, hi)]
        S = dg.assemble(tuple(ns), k, lower=tuple(a * h for a in lo), upper=tuple((b + 1) * h for b in hi))
        xs = np.empty(S.shape[0])
        for cz in range(ns[2]):
            for cy in range(ns[1]):
                for cx in range(ns[0]):
                    s = (cz * ns[1] + cy) * ns[0] + cx
                    g = ((lo[2] + cz) * n + lo[1] + cy) * n + lo[0] + cx
                    xs[s * NV:(s + 1) * NV] = x[g * NV:(g + 1) * NV]
        ys = S @ xs
        t = [c - a for c, a in zip(cell, lo)]
        s = (t[2] * ns[1] + t[1]) * ns[0] + t[0]
        g = (cell[2] * n + cell[1]) * n + cell[0]
        ref = ys[s * NV:(s + 1) * NV]
        assert np.abs(y[g * NV:(g + 1) * NV] - ref).max() <= 1e-12 * np.abs(ref).max(), cell


@pytest.mark.parametrize("case,chunks", [(dict(n_cells=(3, 2, 8), k=2), "4"), (dict(n_cells=(2, 3, 9), k=3), "3"),
                                         (dict(n_cells=(2, 2, 16), k=4), "8"), (dict(n_cells=(2, 2, 3), k=2), "4")],
                         ids=lambda v: v if isinstance(v, str) else _id(v))
def test_dg_pipelined_apply_host(case, chunks, torch, monkeypatch):
    # mf_apply_host by z cell-layer ranges (each range uploads through the layer above it);
    # (2, 2, 3) with 4 ranges takes the unpipelined path
    monkeypatch.setenv("MF_HOST_PIPELINE", chunks)
    A = _ref(case)
    op = _op(case)
    for s in (1, 2):
        x = seeded(A.shape[0], s)
        y = op.apply_host(x)
        assert rel_l2(y, A @ x) <= 1e-12
        y_dev = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        np.testing.assert_array_equal(y, y_dev)  # plain stores: the same bits
