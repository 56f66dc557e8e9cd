"""Host-side DoF numbering of unstructured hex meshes (mf_hex_number_dofs;
SURVEY.md §8(f) f3, R21) against the oracle's brute-force rule (one DoF
per distinct support point).  Numberings are not unique: what must agree is the
partition of cell-local nodes into DoFs (a bijection between the two numberings
consistent over every cell) and the boundary set.  Host code only, no GPU."""
import numpy as np
import pytest

from tests import _hexmesh as hm


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_numbering_matches_coordinate_partition(k, seed):
    from paper_1910_13247_b200 import hex_number_dofs

    m = hm.conforming((3, 2, 2), k, jitter=0.2, seed=seed)
    cd, n, bnd = hex_number_dofs(m["cells"], k)
    assert n == m["n_dofs"]
    mp = -np.ones(n, dtype=np.int64)
    for a, b in zip(cd.reshape(-1), m["cell_dofs"].reshape(-1)):
        assert mp[a] in (-1, b)
        mp[a] = b
    assert len(np.unique(mp)) == n and mp.min() >= 0
    ob = np.zeros(n, dtype=bool)
    ob[m["dirichlet"]] = True
    np.testing.assert_array_equal(bnd, ob[mp])


def test_counts_on_structured_brick():
    from paper_1910_13247_b200 import hex_number_dofs

    for k in (1, 2, 4):
        m = hm.conforming((4, 3, 2), k, jitter=0.0, seed=5)
        _, n, bnd = hex_number_dofs(m["cells"], k)
        assert n == (4 * k + 1) * (3 * k + 1) * (2 * k + 1)
        assert bnd.sum() == n - (4 * k - 1) * (3 * k - 1) * (2 * k - 1)


def test_numbering_errors():
    from paper_1910_13247_b200 import MFError, hex_number_dofs

    cells = np.arange(8, dtype=np.int32)[None, :].copy()
    cells[0, 7] = 0
    with pytest.raises(MFError) as e:
        hex_number_dofs(cells, 2)
    assert e.value.name == "MF_ERR_ARGUMENT"
    # three cells on one face
    c = np.array([[0, 1, 2, 3, 4, 5, 6, 7], [4, 5, 6, 7, 8, 9, 10, 11], [12, 13, 14, 15, 4, 5, 6, 7]],
                 dtype=np.int32)
    with pytest.raises(MFError):
        hex_number_dofs(c, 1)
