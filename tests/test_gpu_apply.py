"""GPU parity of mf_apply / mf_diagonal against the CPU oracle (§8(a) a3-a9).

Element-by-element relative L2 <= 1e-12 (R11) on seeded splitmix vectors,
at sizes spanning several thread blocks with a ragged tail, for every degree,
both dimensions, affine and curved geometry, constant and variable
coefficient, Dirichlet and Neumann; plus the full BASELINE sizes (cfg 3 via
the Kronecker-sum oracle, cfg 4 on sampled rows) in the launch configuration
bench.py times."""
import numpy as np
import pytest

import oracle
from tests._helpers import CUDA_ORACLE_TOL, cuda_operator, oracle_problem, rel_l2, seeded

pytestmark = pytest.mark.gpu

CASES = [
    # BASELINE configs[0]: 2D Q1 on 4x4
    dict(dim=2, n_cells=(4, 4), k=1),
    dict(dim=2, n_cells=(7, 5), k=2, upper=(1.0, 0.6)),
    dict(dim=2, n_cells=(5, 3), k=5, coeff=2.5),
    dict(dim=2, n_cells=(3, 4), k=8),
    dict(dim=2, n_cells=(6, 5), k=3, geometry="sine", coeff="variable"),
    dict(dim=2, n_cells=(9, 7), k=1, dirichlet=0b0101),
    dict(dim=3, n_cells=(5, 4, 3), k=1),
    dict(dim=3, n_cells=(5, 4, 3), k=2, lower=(-0.5, 0.0, 0.2), upper=(1.0, 0.7, 1.0)),
    dict(dim=3, n_cells=(6, 3, 4), k=3, coeff=0.7),
    dict(dim=3, n_cells=(3, 4, 5), k=4),
    dict(dim=3, n_cells=(3, 3, 2), k=5),
    dict(dim=3, n_cells=(3, 2, 2), k=6),
    dict(dim=3, n_cells=(2, 2, 1), k=7),
    dict(dim=3, n_cells=(2, 1, 2), k=8),
    dict(dim=3, n_cells=(5, 4, 3), k=2, dirichlet=0),
    dict(dim=3, n_cells=(4, 4, 4), k=3, dirichlet=0b100110),
    dict(dim=3, n_cells=(4, 3, 3), k=2, coeff="variable"),
    dict(dim=3, n_cells=(4, 4, 3), k=3, geometry="sine"),
    dict(dim=3, n_cells=(4, 3, 4), k=2, geometry="sine", coeff="variable"),
    dict(dim=3, n_cells=(8, 8, 8), k=3, geometry="sine", coeff="variable"),  # cfg 4 shape, small
    dict(dim=3, n_cells=(3, 3, 3), k=4, geometry="sine", coeff="variable", dirichlet=0),
    dict(dim=3, n_cells=(16, 16, 16), k=2),  # cfg 2
    # degenerate meshes: every DoF constrained (A = I), one cell, one-cell-thick plates
    dict(dim=3, n_cells=(1, 1, 1), k=1),
    dict(dim=2, n_cells=(1, 1), k=3, dirichlet=0),
    dict(dim=3, n_cells=(1, 6, 1), k=2, dirichlet=0),
    dict(dim=3, n_cells=(1, 1, 5), k=3, geometry="sine", coeff="variable", dirichlet=0b110000),
]


def _id(c):
    return f"{c['dim']}d-k{c['k']}-{'x'.join(map(str, c['n_cells']))}-{c.get('geometry', 'cart')}-{c.get('coeff', 1.0)}-d{c.get('dirichlet')}"


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_apply_matches_assembled_oracle(case, torch):
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    assert op.n_local == A.n
    seeds = range(1, 11) if case["n_cells"] in ((4, 4), (16, 16, 16), (8, 8, 8)) else range(1, 4)
    for s in seeds:
        x = seeded(A.n, s)
        y_ref = A @ x
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        err = rel_l2(y, y_ref)
        assert err <= CUDA_ORACLE_TOL, (s, err)
    # identity rows are exact
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


TILE_CASES = [
    dict(dim=3, n_cells=(9, 10, 11), k=2),                       # 2x2 ragged tiles, many z-chunks
    dict(dim=3, n_cells=(16, 16, 16), k=2, dirichlet=0),
    dict(dim=3, n_cells=(9, 9, 13), k=3, upper=(1.0, 2.0, 0.5), coeff=3.0),
    dict(dim=3, n_cells=(9, 17, 7), k=4),                        # 3x3 tiles, ragged in x and y
    dict(dim=3, n_cells=(4, 8, 5), k=4, dirichlet=0b011001),
    dict(dim=3, n_cells=(1, 1, 1), k=4),
    dict(dim=3, n_cells=(5, 3, 20), k=4, dirichlet=0),
    dict(dim=3, n_cells=(17, 1, 1), k=2, dirichlet=0),           # one-cell-thick in y and z
    dict(dim=3, n_cells=(1, 5, 9), k=3, dirichlet=0b000011),
]


@pytest.mark.parametrize("variant", ["general", "plane", "halo"])
@pytest.mark.parametrize("case", TILE_CASES, ids=_id)
def test_cartesian_variants_match_oracle(case, variant, torch):
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    if variant == "halo" and not (case["k"] == 4 and (case["n_cells"][0] % 32 or case.get("dirichlet") is None
                                                       or case["dirichlet"] & 2)
                                  and (case["n_cells"][1] % 2 or case.get("dirichlet") is None or case["dirichlet"] & 8)):
        pytest.skip("outside the halo kernel's domain (k = 4, Dirichlet x+ / y+ on full last tiles)")
    op.set_variant(variant)
    assert op.info()["apply_variant"] == {"general": 1, "plane": 3, "halo": 6}[variant]
    for s in (1, 2, 3):
        x = seeded(A.n, s)
        y_ref = A @ x
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, y_ref) <= CUDA_ORACLE_TOL, (s, rel_l2(y, y_ref))
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


ZSPLIT_CASES = [
    (dict(dim=3, n_cells=(9, 10, 11), k=2), "plane"),
    (dict(dim=3, n_cells=(9, 17, 7), k=4, dirichlet=0b011001), "plane"),
    (dict(dim=3, n_cells=(5, 3, 20), k=4, dirichlet=0), "plane"),
    (dict(dim=3, n_cells=(4, 4, 1), k=3), "plane"),
    (dict(dim=3, n_cells=(4, 4, 2), k=3), "plane"),
    (dict(dim=3, n_cells=(4, 4, 3), k=3), "plane"),
    (dict(dim=3, n_cells=(6, 5, 7), k=3, geometry="sine", coeff="variable"), "auto"),
    (dict(dim=3, n_cells=(3, 3, 2), k=5), "auto"),
    (dict(dim=3, n_cells=(5, 4, 6), k=2, coeff="variable"), "general"),
    (dict(dim=3, n_cells=(5, 4, 1), k=2), "general"),
]


@pytest.mark.parametrize("case,variant", ZSPLIT_CASES, ids=lambda v: v if isinstance(v, str) else _id(v))
def test_zsplit_launch_sequence_matches_oracle(case, variant, torch, monkeypatch):
    # the multi-GPU overlap order (boundary cell layers, then the interior; §8(e)) run on
    # one GPU without the exchange: MF_ZSPLIT=1
    monkeypatch.setenv("MF_ZSPLIT", "1")
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    op.set_variant(variant)
    for s in (1, 2):
        x = seeded(A.n, s)
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, A @ x) <= CUDA_ORACLE_TOL, (s, rel_l2(y, A @ x))
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


@pytest.mark.parametrize("case", CASES[::2], ids=_id)
def test_diagonal_matches_assembled_oracle(case, torch):
    p = oracle_problem(case)
    d_ref = oracle.CSR(p).diagonal()
    d = cuda_operator(case).diagonal().cpu().numpy()
    assert np.abs(d - d_ref).max() <= 1e-12 * np.abs(d_ref).max()
    assert np.all(d > 0)


@pytest.mark.parametrize("geometry,coeff", [("cartesian", 1.0), ("sine", 1.0), ("sine", "variable")])
def test_neumann_kernel_on_gpu(geometry, coeff, torch):
    case = dict(dim=3, n_cells=(5, 4, 4), k=3, geometry=geometry, coeff=coeff, dirichlet=0)
    op = cuda_operator(case)
    one = torch.ones(op.n_local, dtype=torch.float64, device="cuda")
    y = op.apply(one)
    d = op.diagonal()
    assert y.abs().max().item() <= 1e-13 * d.abs().max().item() * 8


def test_zero_and_linearity(torch):
    case = dict(dim=3, n_cells=(4, 4, 4), k=4)
    op = cuda_operator(case)
    z = op.apply(op.new_vector())
    assert z.abs().max().item() == 0.0
    x = torch.from_numpy(seeded(op.n_local, 1)).cuda()
    y = torch.from_numpy(seeded(op.n_local, 2)).cuda()
    lhs = op.apply(2.0 * x - 3.0 * y)
    rhs = 2.0 * op.apply(x) - 3.0 * op.apply(y)
    assert ((lhs - rhs).norm() / rhs.norm()).item() < 1e-14


def test_symmetry_on_gpu(torch):
    case = dict(dim=3, n_cells=(4, 3, 5), k=3, geometry="sine", coeff="variable")
    op = cuda_operator(case)
    x = torch.from_numpy(seeded(op.n_local, 4)).cuda()
    y = torch.from_numpy(seeded(op.n_local, 5)).cuda()
    a = torch.dot(x, op.apply(y)).item()
    b = torch.dot(y, op.apply(x)).item()
    assert abs(a - b) <= 1e-13 * x.norm().item() * y.norm().item()


def test_apply_host_matches_device(torch):
    case = dict(dim=3, n_cells=(6, 5, 4), k=4)
    op = cuda_operator(case)
    x = seeded(op.n_local, 7)
    y_dev = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    y_host = op.apply_host(x)
    np.testing.assert_array_equal(y_dev.shape, y_host.shape)
    assert rel_l2(y_host, y_dev) < 1e-15


HOST_PIPELINE_CASES = [
    (dict(dim=3, n_cells=(9, 10, 11), k=2), "4", "plane"),                # ragged ranges (3,3,3,2 layers)
    (dict(dim=3, n_cells=(6, 5, 16), k=4), "4", "plane"),
    (dict(dim=3, n_cells=(6, 5, 16), k=4, dirichlet=0), "3", "plane"),
    (dict(dim=3, n_cells=(9, 17, 13), k=3, dirichlet=0b011001), "5", "plane"),
    (dict(dim=3, n_cells=(5, 3, 20), k=4, dirichlet=0b110000), "2", "plane"),
    (dict(dim=3, n_cells=(4, 4, 8), k=3), "4", "plane"),                   # two layers per range
    (dict(dim=3, n_cells=(4, 4, 16), k=3), "8", "plane"),
    (dict(dim=3, n_cells=(5, 4, 11), k=3, geometry="sine", coeff="variable"), "4", "auto"),
    (dict(dim=3, n_cells=(3, 4, 9), k=5, dirichlet=0b100110), "3", "auto"),
    (dict(dim=3, n_cells=(6, 5, 8), k=2, coeff="variable", dirichlet=0), "4", "general"),
    (dict(dim=3, n_cells=(6, 5, 16), k=4), "8", "general"),
]


@pytest.mark.parametrize("case,chunks,variant", HOST_PIPELINE_CASES,
                         ids=lambda v: v if isinstance(v, str) else _id(v))
def test_pipelined_apply_host_matches_oracle(case, chunks, variant, torch, monkeypatch):
    # mf_apply_host overlaps the copies with the apply by z cell-layer ranges
    monkeypatch.setenv("MF_HOST_PIPELINE", chunks)
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    op.set_variant(variant)
    for s in (1, 2, 3):
        x = seeded(A.n, s)
        y = op.apply_host(x)
        assert rel_l2(y, A @ x) <= CUDA_ORACLE_TOL, (s, rel_l2(y, A @ x))
        y_dev = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, y_dev) <= 1e-14
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


def test_length_and_argument_errors(torch):
    from paper_1910_13247_b200 import MFError

    op = cuda_operator(dict(dim=3, n_cells=(2, 2, 2), k=2))
    x = op.new_vector()
    with pytest.raises(MFError) as e:
        op.apply(x[:-1])
    assert e.value.name == "MF_ERR_LENGTH"
    with pytest.raises(MFError) as e:
        op.apply(x, x)
    assert e.value.name == "MF_ERR_ARGUMENT"
    with pytest.raises(MFError) as e:
        cuda_operator(dict(dim=3, n_cells=(2, 2, 2), k=3, geometry="sine", eps=2.0))
    assert e.value.name == "MF_ERR_SINGULAR"


def test_cfg3_full_size_vs_kronecker_oracle(torch):
    # BASELINE configs[2]: Q4 on 64^3 (16,974,593 DoFs), the bench workload, auto variant
    case = dict(dim=3, n_cells=(64, 64, 64), k=4)
    p = oracle_problem(case)
    op = cuda_operator(case)
    x = seeded(op.n_local, 1)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    y_ref = oracle.kron_apply(p, x)
    assert rel_l2(y, y_ref) <= CUDA_ORACLE_TOL
    rows = np.random.default_rng(0).choice(op.n_local, 200, replace=False)
    np.testing.assert_allclose(y[rows], oracle.apply_rows(p, rows, x), rtol=0,
                               atol=1e-12 * np.abs(y_ref).max())


def test_cfg4_full_size_sampled_rows(torch):
    # BASELINE configs[3]: Q3 on the deformed 64^3 cube, variable coefficient, stored metric
    case = dict(dim=3, n_cells=(64, 64, 64), k=3, geometry="sine", coeff="variable")
    p = oracle_problem(case)
    op = cuda_operator(case)
    x = seeded(op.n_local, 1)
    y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    rng = np.random.default_rng(1)
    rows = np.concatenate([rng.choice(op.n_local, 300, replace=False), [0, op.n_local - 1, op.n_local // 2]])
    ref = oracle.apply_rows(p, rows, x)
    assert np.abs(y[rows] - ref).max() <= CUDA_ORACLE_TOL * np.abs(ref).max()


@pytest.mark.parametrize("nc", [32, 64])
def test_cfg4_full_vector_vs_assembled_csr(nc, torch):
    # BASELINE configs[3] operator (Q3, deformed cube, variable c, stored metric) over EVERY DoF
    # against the assembled CSR oracle in the bench launch configuration (auto variant): 32^3
    # (1.3 GB CSR) always, 64^3 (10.7 GB CSR, the bench size) when the host has the memory
    import psutil

    need = 1.4e9 if nc == 32 else 2.5e10
    if psutil.virtual_memory().available < need:
        pytest.skip(f"host memory below {need / 1e9:.0f} GB for the {nc}^3 CSR")
    case = dict(dim=3, n_cells=(nc, nc, nc), k=3, geometry="sine", coeff="variable")
    p = oracle_problem(case)
    A = oracle.CSR(p)
    op = cuda_operator(case)
    assert op.n_local == A.n
    for s in (1, 2):
        x = seeded(A.n, s)
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        y_ref = A @ x
        assert rel_l2(y, y_ref) <= CUDA_ORACLE_TOL, (s, rel_l2(y, y_ref))
    m = oracle.constrained_mask_fast(p)
    np.testing.assert_array_equal(y[m], x[m])


def test_cfg4_full_size_energy_of_linears(torch):
    # BASELINE configs[3] geometry and coefficient (Q3, deformed 64^3, variable c) under Neumann:
    # u_a^T A u_b = delta_ab int c dx for the physical linears u_a = x_a (the property
    # tests/test_oracle_operator.py::test_deformed_variable_coefficient_energy_of_linears pins
    # on the oracle), checked at full size where the oracle cannot assemble
    from tests.test_oracle_operator import _integral_of_c_unit_cube, _node_coords

    case = dict(dim=3, n_cells=(64, 64, 64), k=3, geometry="sine", coeff="variable", dirichlet=0)
    p = oracle_problem(case)
    op = cuda_operator(case)
    X = torch.from_numpy(_node_coords(p, physical=True)).cuda()
    AX = [op.apply(X[:, b].contiguous()) for b in range(3)]
    G = np.array([[torch.dot(X[:, a], AX[b]).item() for b in range(3)] for a in range(3)])
    Ic = _integral_of_c_unit_cube()
    assert np.abs(G - G[0, 0] * np.eye(3)).max() <= 1e-11 * Ic
    assert abs(G[0, 0] - Ic) <= 1e-7 * Ic


def _one_d(k, n, which):
    # global 1D stiffness (which=0) / mass (which=1) on [0,1] from the oracle, no constraints
    return oracle.CSR(oracle.problem(dim=1, n_cells=(n,), degree=k), which=which, dirichlet=False).dense()


@pytest.mark.parametrize("cfg", [((256, 256, 256), 4), ((256, 256, 256), 6)], ids=["cfg5q4", "cfg5q6"])
def test_full_size_separable_input(cfg, torch):
    # BASELINE configs[4] sizes on ONE GPU (1.08 / 3.63 billion DoFs; 64-bit indexing):
    # x = a (x) b (x) c with a, b, c vanishing at the ends, so on the brick
    # A x = (K a)(M b)(M c) + (M a)(K b)(M c) + (M a)(M b)(K c) with the oracle's 1D
    # matrices (the Kronecker identity is pinned in tests/test_oracle_operator.py);
    # checked row by row at sampled DoFs, and over all DoFs with torch outer products
    (nc, k) = cfg
    n1 = k * nc[0] + 1
    K1, M1 = _one_d(k, nc[0], 0), _one_d(k, nc[0], 1)
    v = [seeded(n1, s) for s in (21, 22, 23)]
    for w in v:
        w[0] = w[-1] = 0.0
    Kv, Mv = [K1 @ w for w in v], [M1 @ w for w in v]
    for w in Kv + Mv:  # Dirichlet rows are identity rows and x vanishes there
        w[0] = w[-1] = 0.0
    op = cuda_operator(dict(dim=3, n_cells=nc, k=k))
    assert op.n_local == n1 ** 3
    g = [torch.from_numpy(w).cuda() for w in v]
    x = torch.einsum("k,j,i->kji", g[2], g[1], g[0]).reshape(-1)  # z slowest, x fastest
    y = op.apply(x)
    del x
    rows = np.random.default_rng(2).integers(0, op.n_local, 300)
    yr = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    i, j, kk = rows % n1, (rows // n1) % n1, rows // (n1 * n1)
    ref = Kv[0][i] * Mv[1][j] * Mv[2][kk] + Mv[0][i] * Kv[1][j] * Mv[2][kk] + Mv[0][i] * Mv[1][j] * Kv[2][kk]
    scale = np.abs(ref).max()
    assert np.abs(yr - ref).max() <= CUDA_ORACLE_TOL * scale
    t = [torch.from_numpy(a).cuda() for a in (Kv[0], Mv[0], Kv[1], Mv[1], Kv[2], Mv[2])]
    exp = torch.einsum("k,j,i->kji", t[5], t[3], t[0]).reshape(-1)
    exp += torch.einsum("k,j,i->kji", t[5], t[2], t[1]).reshape(-1)
    exp += torch.einsum("k,j,i->kji", t[4], t[3], t[1]).reshape(-1)
    err = ((y - exp).norm() / exp.norm()).item()
    assert err <= CUDA_ORACLE_TOL, err
