"""GPU parity of the unstructured-hex operator (mf_create_hex)
against the pinned oracle (oracle/hex.py): jittered trilinear meshes with rotated
cell frames and shuffled vertex numbers, DoFs numbered by the oracle (coordinates)
or by the library (mf_hex_number_dofs, compared through the coordinate bijection),
constant / variable coefficient, Dirichlet / Neumann, the 2:1 hanging interface
through constraint lines in the gather / scatter, diagonal, Chebyshev-PCG."""
import numpy as np
import pytest

import synth
from oracle import hex as ohex
from oracle import solvers
from tests import _hexmesh as hm
from tests._helpers import CUDA_ORACLE_TOL, rel_l2, seeded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def _op(m, coeff=1.0, dirichlet=True):
    from paper_1910_13247_b200 import HexOperator

    return HexOperator(m["vertices"], m["cells"], m["k"], m["cell_dofs"], m["n_dofs"], m["lines"],
                       m["dirichlet"] if dirichlet else (), coeff=coeff)


CASES = [
    dict(n_cells=(3, 2, 2), k=1, jitter=0.2),
    dict(n_cells=(3, 2, 2), k=2, jitter=0.25),
    dict(n_cells=(2, 3, 2), k=3, jitter=0.2, coeff="variable"),
    dict(n_cells=(2, 2, 2), k=4, jitter=0.2),
    dict(n_cells=(2, 2, 1), k=5, jitter=0.15),
    dict(n_cells=(2, 1, 1), k=6, jitter=0.1, coeff="variable"),
    dict(n_cells=(7, 5, 6), k=3, jitter=0.2),     # several blocks and a ragged tail
    dict(n_cells=(3, 3, 2), k=2, jitter=0.0),     # rotated frames on the plain brick
]


def _id(c):
    return f"k{c['k']}-{'x'.join(map(str, c['n_cells']))}-j{c['jitter']}-{c.get('coeff', 1.0)}"


@pytest.mark.parametrize("case", CASES, ids=_id)
@pytest.mark.parametrize("dirichlet", [True, False])
def test_apply_matches_oracle(case, dirichlet, torch):
    coeff = case.get("coeff", 1.0)
    m = hm.conforming(case["n_cells"], case["k"], jitter=case["jitter"], seed=case["k"])
    A = hm.oracle_matrix(m, coeff="variable" if coeff == "variable" else "constant",
                         value=1.0 if coeff == "variable" else coeff, dirichlet=dirichlet)
    op = _op(m, coeff, dirichlet)
    assert op.info()["apply_variant"] == 5
    for s in (1, 2):
        x = seeded(m["n_dofs"], s)
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, A @ x) <= CUDA_ORACLE_TOL, (s, rel_l2(y, A @ x))
    if dirichlet:
        np.testing.assert_array_equal(y[m["dirichlet"]], x[m["dirichlet"]])
    d = op.diagonal().cpu().numpy()
    assert np.abs(d - A.diagonal()).max() <= 1e-12 * np.abs(A.diagonal()).max()
    yh = op.apply_host(x)
    assert rel_l2(yh, A @ x) <= CUDA_ORACLE_TOL


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_library_numbering_matches_oracle(k, torch):
    from paper_1910_13247_b200 import hex_number_dofs

    m = hm.conforming((3, 3, 2), k, jitter=0.2, seed=20 + k)
    cd, n, bnd = hex_number_dofs(m["cells"], k)
    mp = np.empty(n, dtype=np.int64)  # library DoF -> oracle DoF
    mp[cd.reshape(-1)] = m["cell_dofs"].reshape(-1)
    lib = dict(m, cell_dofs=cd, dirichlet=np.nonzero(bnd)[0])
    A = hm.oracle_matrix(m)
    op = _op(lib)
    x_or = seeded(n, 4)
    y = op.apply(torch.from_numpy(x_or[mp]).cuda()).cpu().numpy()
    assert rel_l2(y, (A @ x_or)[mp]) <= CUDA_ORACLE_TOL


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_hanging_constraints_in_gather_scatter(k, torch):
    m = hm.two_block((2, 2, 1), 2, k)
    A = hm.oracle_matrix(m)
    op = _op(m)
    for s in (1, 2):
        x = seeded(m["n_dofs"], s)
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, A @ x) <= CUDA_ORACLE_TOL
    d = op.diagonal().cpu().numpy()
    assert np.abs(d - A.diagonal()).max() <= 1e-12 * np.abs(A.diagonal()).max()


@pytest.mark.parametrize("case", [dict(n_cells=(4, 3, 3), k=2), dict(n_cells=(2, 2, 2), k=4)],
                         ids=lambda c: f"k{c['k']}")
def test_chebyshev_pcg_matches_oracle(case, torch):
    m = hm.conforming(case["n_cells"], case["k"], jitter=0.2, seed=9)
    A = hm.oracle_matrix(m)
    n = m["n_dofs"]
    mask = np.zeros(n, dtype=bool)
    mask[m["dirichlet"]] = True
    s = synth.with_zero_dirichlet(synth.vector(n, 0), mask)
    b = synth.with_zero_dirichlet(seeded(n, 11), mask)
    ref = solvers.chebyshev_pcg(A.dot, A.diagonal(), b, s, rel_tol=1e-10)
    op = _op(m)
    x, res = op.cg_solve(torch.from_numpy(b).cuda(), rel_tol=1e-10)
    assert abs(res.lambda_max - ref.lambda_max) <= 1e-9 * ref.lambda_max
    assert abs(res.iterations - ref.iterations) <= 1
    assert rel_l2(x.cpu().numpy(), ref.x) <= 1e-8


def test_hex_errors(torch):
    from paper_1910_13247_b200 import MFError

    m = hm.conforming((2, 2, 2), 2, jitter=0.0, seed=1)
    bad = dict(m, cells=m["cells"][:, [1, 0, 3, 2, 5, 4, 7, 6]])  # mirrored frame: det J < 0
    with pytest.raises(MFError) as e:
        _op(bad)
    assert e.value.name == "MF_ERR_SINGULAR"
    cd = m["cell_dofs"].copy()
    cd[0, 0] = m["n_dofs"]
    with pytest.raises(MFError) as e:
        _op(dict(m, cell_dofs=cd))
    assert e.value.name == "MF_ERR_ARGUMENT"
    cd[0, 0] = -5  # no constraint lines
    with pytest.raises(MFError) as e:
        _op(dict(m, cell_dofs=cd))
    assert e.value.name == "MF_ERR_ARGUMENT"


def _support_coords(V, C, cd, n, k):
    """Physical coordinates of every DoF (trilinear map of the GLL nodes), test-side numpy."""
    import oracle

    nodes = oracle.gll(k)
    N = k + 1
    loc = np.array([[i % N, (i // N) % N, i // (N * N)] for i in range(N ** 3)])
    xi = nodes[loc]  # [nv][3]
    corners = np.array([[v & 1, (v >> 1) & 1, v >> 2] for v in range(8)], dtype=np.float64)
    Nv = np.prod(np.where(corners[None, :, :] == 1, xi[:, None, :], 1.0 - xi[:, None, :]), axis=2)  # [nv][8]
    X = np.einsum("lv,cvd->cld", Nv, V[C])  # [cells][nv][3]
    coords = np.empty((n, 3))
    coords[cd.reshape(-1)] = X.reshape(-1, 3)
    return coords


def test_full_size_hex3_properties(torch):
    """bench.py's hex3 mesh (64^3 jittered, rotated, library numbering) at full size: the
    Neumann kernel, physical linears (interior rows vanish, Galerkin exactness on trilinear
    cells), and symmetry with the variable coefficient (R5), in the launch configuration
    bench.py times."""
    from paper_1910_13247_b200 import HexOperator, hex_number_dofs

    V, C = synth.hex_mesh((64, 64, 64), jitter=0.2, seed=0)
    k = 3
    cd, n, bnd = hex_number_dofs(C, k)
    assert n == 193 ** 3
    op = HexOperator(V, C, k, cd, n)  # Neumann, c = 1
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    d = op.diagonal()
    assert op.apply(one).abs().max().item() <= 1e-12 * d.abs().max().item()
    coords = _support_coords(V, C, cd, n, k)
    u = torch.from_numpy(coords @ np.array([0.3, -1.1, 0.7]) + 0.4).cuda()
    y = op.apply(u).cpu().numpy()
    interior = ~bnd
    assert np.abs(y[interior]).max() <= 1e-11 * d.abs().max().item()
    assert np.abs(y[bnd]).max() > 1e-6
    # variable coefficient under Neumann: u_a^T A u_b = delta_ab int c dx for the physical
    # linears (pinned on the oracle by test_oracle_hex.py::
    # test_variable_coefficient_energy_of_linears_on_jittered_mesh)
    from tests.test_oracle_operator import _integral_of_c_unit_cube

    op = HexOperator(V, C, k, cd, n, coeff="variable")
    X = torch.from_numpy(coords).cuda()
    AX = [op.apply(X[:, j].contiguous()) for j in range(3)]
    G = np.array([[torch.dot(X[:, i], AX[j]).item() for j in range(3)] for i in range(3)])
    Ic = _integral_of_c_unit_cube()
    assert np.abs(G - G[0, 0] * np.eye(3)).max() <= 1e-11 * Ic
    assert abs(G[0, 0] - Ic) <= 1e-6 * Ic
    op = HexOperator(V, C, k, cd, n, dirichlet=np.nonzero(bnd)[0], coeff="variable")
    a = torch.from_numpy(seeded(n, 1)).cuda()
    b = torch.from_numpy(seeded(n, 2)).cuda()
    lhs, rhs = torch.dot(a, op.apply(b)).item(), torch.dot(b, op.apply(a)).item()
    assert abs(lhs - rhs) <= 1e-12 * a.norm().item() * b.norm().item() * d.abs().max().item()
