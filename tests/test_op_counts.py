"""Closed-form SolveReport.ops tallies against the reference's own CounterBox
counts (golden vectors made by running bandix, tests/golden/make_golden.py).
CPU only."""
import numpy as np

from paper_1804_09666_b200.inverse import _sip_hb_ops


def _tuple(c):
    return [int(c.adds), int(c.subs), int(c.muls), int(c.divs)]


def test_sip_hb_dense_ops_match_reference(golden):
    """sip_hb_solve(mode="dense"): 4N^2 + 20N - 24 per iteration (the dense
    applies, inverse.py:198-202), not SIP's 31N - 36."""
    g = golden("inverse")
    n = g["hb_main"].shape[1]
    for s in range(g["hb_k"].shape[0]):
        assert _tuple(_sip_hb_ops(n, int(g["hb_k"][s]))) == g["hb_ops"][s].tolist()
        assert sum(g["hb_ops"][s]) == (4 * n * n + 20 * n - 24) * int(g["hb_k"][s])


def test_sip_hb_banded_ops_match_reference(golden):
    """sip_hb_solve(mode="banded", hb_bandwidth=32): band applies
    (inverse.py:48-61) -- the converging explicit-width case."""
    g = golden("hbband")
    n = g["hbb_main"].shape[1]
    for s in range(2):
        key = f"sip_{s}_32"
        assert int(g[key + "_st"]) == 0
        ops = _sip_hb_ops(n, int(g[key + "_k"]), "banded", 32, 32)
        assert _tuple(ops) == g[key + "_ops"].tolist()


def test_sip_hb_ops_vectorised():
    k = np.array([3, 5])
    c = _sip_hb_ops(100, k, "banded", np.array([2, 4]), np.array([4, 8]))
    assert c.muls.tolist() == [_sip_hb_ops(100, 3, "banded", 2, 4).muls, _sip_hb_ops(100, 5, "banded", 4, 8).muls]
