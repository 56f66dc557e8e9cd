"""Full-size parity with a seeded random (non-separable) input, BASELINE configs[4] on one GPU
in the launch configuration bench.py times (§8(a) a3-a7; R11: 1e-12): the 256^3-cell cube with
Q6 (k_apply_tc, 3.63 B DoFs) and Q4 (k_apply_halo, 1.08 B DoFs).

The input is synth's counter-based splitmix64 vector, generated on the GPU by the same
arithmetic in torch (checked bit for bit against synth on two slices).  The oracle evaluates
sampled rows one by one (oracle.apply_rows: the cells around the node, brute-force quadrature),
which reads x only on those cells' nodes: its host vector is a lazily allocated zero array
(untouched pages cost no memory) filled with synth values on each sampled row's neighbourhood.
Rows are drawn at random plus structural ones (mesh corners, edges, the Dirichlet faces, vertex
planes and cell-interior planes)."""
import numpy as np
import pytest

import oracle
import synth
from tests._helpers import CUDA_ORACLE_TOL, cuda_operator, oracle_problem

pytestmark = pytest.mark.gpu

SEED = 31
_GOLD, _M1, _M2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _s64(v):  # the uint64 constant as a two's-complement int64
    return v - (1 << 64) if v >= 1 << 63 else v


def _lsr(torch, z, s):  # logical right shift of int64
    return (z >> s) & ((1 << (64 - s)) - 1)


def _uniform_cuda(torch, out, first, seed):
    """synth.uniform(first, len(out), seed) computed on the GPU into `out` (chunked)."""
    n, ch = out.numel(), 1 << 27
    for a in range(0, n, ch):
        b = min(n, a + ch)
        z = torch.arange(first + a, first + b, dtype=torch.int64, device=out.device) + seed * (1 << 40)
        z = z + _s64(_GOLD)
        z = (z ^ _lsr(torch, z, 30)) * _s64(_M1)
        z = (z ^ _lsr(torch, z, 27)) * _s64(_M2)
        z = z ^ _lsr(torch, z, 31)
        out[a:b] = 2.0 * (_lsr(torch, z, 11).to(torch.float64) * (1.0 / 9007199254740992.0)) - 1.0
        del z


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _rows(n1, k, rng, m=160):
    r = list(rng.integers(0, n1 ** 3, m))
    for (x, y, z) in [(1, 1, 1), (n1 - 2, n1 - 2, n1 - 2), (k, 1, 1), (k, k, k), (n1 // 2, k, n1 - 2),
                      (0, 5, 7), (3, 0, 9), (n1 - 1, 4, 4), (2 * k, 2 * k + 1, 2 * k + 2), (k + 1, n1 // 3, k * 7)]:
        r.append(z * n1 * n1 + y * n1 + x)
    return np.array(sorted(set(int(v) for v in r)), dtype=np.int64)


def _host_x(n, n1, k, rows):
    """zeros except the synth values on every sampled row's cell neighbourhood"""
    x = np.zeros(n)
    for g in rows:
        m = (g % n1, (g // n1) % n1, g // (n1 * n1))
        lo = [max(0, (mi // k - (1 if mi % k == 0 else 0)) * k) for mi in m]
        hi = [min(n1 - 1, (mi // k + 1) * k) for mi in m]
        for zz in range(lo[2], hi[2] + 1):
            for yy in range(lo[1], hi[1] + 1):
                first = zz * n1 * n1 + yy * n1 + lo[0]
                x[first:first + hi[0] - lo[0] + 1] = synth.uniform(first, hi[0] - lo[0] + 1, SEED)
    return x


@pytest.mark.parametrize("k", [6, 4], ids=["cfg5q6", "cfg5q4"])
def test_full_size_random_input_sampled_rows(k, torch):
    case = dict(dim=3, n_cells=(256, 256, 256), k=k)
    op = cuda_operator(case)
    n1 = k * 256 + 1
    n = op.n_local
    assert n == n1 ** 3
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    _uniform_cuda(torch, x, 0, SEED)
    for first in (0, n - 1000):  # the GPU generator is synth's, bit for bit
        np.testing.assert_array_equal(x[first:first + 1000].cpu().numpy(), synth.uniform(first, 1000, SEED))
    y = op.apply(x)
    del x
    rows = _rows(n1, k, np.random.default_rng(5))
    yr = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    del y
    ref = oracle.apply_rows(oracle_problem(case), rows, _host_x(n, n1, k, rows))
    scale = np.abs(ref).max()
    err = np.abs(yr - ref).max() / scale
    assert err <= CUDA_ORACLE_TOL, err
