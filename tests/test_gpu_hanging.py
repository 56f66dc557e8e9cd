"""GPU parity of the hanging-node apply (two-block 2:1 interface)
against oracle/hanging.py: relative L2 <= 1e-12 (R11), identity rows exact."""
import numpy as np
import pytest

from oracle import hanging
from tests._helpers import rel_l2, seeded

pytestmark = pytest.mark.gpu

CASES = [
    dict(nc=(2, 2, 1), nzf=2, k=1),
    dict(nc=(3, 2, 2), nzf=3, k=2),
    dict(nc=(2, 3, 2), nzf=1, k=3, upper=(1.0, 2.0, 1.5), z_mid=0.7),
    dict(nc=(4, 4, 2), nzf=4, k=4),
    dict(nc=(1, 2, 1), nzf=2, k=5),
    dict(nc=(8, 8, 4), nzf=8, k=2),
]


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"k{c['k']}-{'x'.join(map(str, c['nc']))}-f{c['nzf']}")
def test_hanging_apply_matches_oracle(c):
    import torch

    from paper_1910_13247_b200 import HangingNodeOperator

    up = c.get("upper", (1.0, 1.0, 1.0))
    zm = c.get("z_mid", 0.5)
    T = hanging.build(c["nc"], c["nzf"], c["k"], upper=up, z_mid=zm)
    A = hanging.operator(T)
    op = HangingNodeOperator(c["nc"], c["nzf"], c["k"], upper=up, z_mid=zm)
    assert op.n_local == T.n
    for s in (1, 2, 3):
        x = seeded(T.n, s)
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, A @ x) <= 1e-12, (s, rel_l2(y, A @ x))
    np.testing.assert_array_equal(y[T.mask], x[T.mask])
