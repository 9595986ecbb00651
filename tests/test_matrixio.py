"""Text matrix I/O (matrixio.py) against the reference's own parser/serializer
outputs (tests/golden/matrixio.json, made by tests/golden/make_golden.py)."""

import json
import os
from fractions import Fraction

import pytest

from paper_1804_09666_b200 import errors
from paper_1804_09666_b200.matrixio import parse_band_text, serialize_band

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "matrixio.json")))


def dec(v):
    return Fraction(v[1], v[2]) if v[0] == "F" else float.fromhex(v[1])


def same(a, b):
    return type(a) is type(b) and a == b


@pytest.mark.parametrize("case", CASES, ids=[f"c{i}" for i in range(len(CASES))])
def test_parse_matches_reference(case):
    if "error" in case:
        with pytest.raises(getattr(errors, case["error"])) as e:
            parse_band_text(case["text"])
        assert str(e.value) == case["message"]
        return
    kind, n, diags, rhs, exact = parse_band_text(case["text"])
    assert (kind, n, exact) == (case["kind"], case["n"], case["exact"])
    ref = [[dec(v) for v in d] for d in case["diags"]]
    assert all(same(a, b) for da, db in zip(diags, ref) for a, b in zip(da, db))
    if case["rhs"] is None:
        assert rhs is None
    else:
        assert all(same(a, dec(b)) for a, b in zip(rhs, case["rhs"]))
        assert isinstance(rhs, tuple) == exact
    assert serialize_band(kind, n, diags, rhs) == case["serialized"]


def test_round_trip_floats():
    diags = [[0.1, -2.5e-300], [1.0, 3.0, 7.25], [1 / 3, float("1e300")]]
    text = serialize_band("tri", 3, diags, [1.0, 2.0, 3.0])
    kind, n, back, rhs, exact = parse_band_text(text)
    assert (kind, n, exact) == ("tri", 3, False)
    assert back == diags and rhs == [1.0, 2.0, 3.0]


@pytest.mark.gpu
def test_parse_to_gpu_container_and_solve(cuda, golden):
    """SPEC.md:161 hand case through the text format and the GPU NTDM."""
    import numpy as np
    from paper_1804_09666_b200 import solve_ntdm
    from paper_1804_09666_b200.matrixio import parse_matrix_text, serialize_matrix
    m, rhs = parse_matrix_text(CASES[0]["text"])
    assert m.exact and isinstance(rhs, tuple)
    rep = solve_ntdm(m, [float(v) for v in rhs])
    assert np.array_equal(rep.x, golden("direct")["ntdm_spec_x"][0])
    assert serialize_matrix(m, [float(v) for v in rhs]).startswith("tri 3\n-1.0 -1.0\n")
