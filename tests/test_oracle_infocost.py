"""Pins of the oracle's orientation factor O(x) and information cost c_I (P:256-269,
SPEC S:238-246)."""
import math

import numpy as np
import pytest

import oracle
from conftest import read_golden

SPEC = {}
for row in read_golden("spec_examples.txt"):
    k, *v = row.split()
    SPEC.setdefault(k, []).append([float(x) for x in v])

CUT30 = math.cos(math.radians(30.0))


def axis_at(theta_deg):
    """Unit axis at angle theta from +x (ideal direction for pos 0 -> PoI (5,0,0))."""
    t = math.radians(theta_deg)
    return [math.cos(t), math.sin(t), 0.0]


def test_orientation_factor_spec_examples():
    poi = [5.0, 0.0, 0.0]
    assert oracle.orientation_factor([0, 0, 0], [1, 0, 0], poi, CUT30) == SPEC["of_aligned"][0][0]
    assert oracle.orientation_factor([0, 0, 0], axis_at(89.0), poi, CUT30) == SPEC["of_outside"][0][0]
    assert oracle.orientation_factor([0, 0, 0], axis_at(20.0), poi, CUT30) == pytest.approx(SPEC["of_twenty"][0][0],
                                                                                           abs=1e-14)


def test_orientation_factor_invariances():
    """invariant under positive scaling of (poi - position); axis length irrelevant;
    the cut is exactly at theta_cut."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        pos = rng.normal(size=3); poi = pos + rng.normal(size=3) * 3
        ax = rng.normal(size=3)
        a = oracle.orientation_factor(pos, ax, poi, 0.2)
        b = oracle.orientation_factor(pos, ax * 7.5, pos + (poi - pos) * 4.0, 0.2)
        assert a == pytest.approx(b, abs=1e-14)
        c = np.dot(ax, poi - pos) / np.linalg.norm(ax) / np.linalg.norm(poi - pos)
        assert a == pytest.approx(c if c >= 0.2 else 0.0, abs=1e-14)
    with pytest.raises(oracle.OracleError):
        oracle.orientation_factor([1, 1, 1], [1, 0, 0], [1, 1, 1], 0.5)


def test_info_cost_closed_forms():
    """c_I = sum_k w_I/(O G + eps): w_I = 0 -> 0; O = 0 -> w_I/eps per pose (the
    barrier peaks); single perspective -> G = its gain."""
    eps = SPEC["info_eps"][0][0]
    entries = [([[0.0, 0.0, 0.0]], [2.5])]
    poi = [0.0, 0.0, 0.0]
    pos = np.array([[3.0, 0, 0], [0, 4.0, 0], [0, 0, -2.0], [1.0, 1.0, 0]])
    axis = np.array([[-1.0, 0, 0], [0, -1.0, 0], [0, 0, 1.0], [1.0, 1.0, 0]])   # last looks away
    o, g, c = oracle.info_cost(entries, pos, axis, 2, poi, CUT30, w_i=25.0, eps=eps)
    assert list(o) == [1.0, 1.0, 1.0, 0.0]
    assert np.allclose(g, 2.5, rtol=1e-15)
    assert c[0] == pytest.approx(2 * 25.0 / (2.5 + eps), rel=1e-15)
    assert c[1] == pytest.approx(25.0 / (2.5 + eps) + 25.0 / eps, rel=1e-15)
    _, _, c0 = oracle.info_cost(entries, pos, axis, 2, poi, CUT30, w_i=0.0, eps=eps)
    assert (c0 == 0).all()
