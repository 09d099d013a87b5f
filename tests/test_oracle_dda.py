"""Pins of the oracle's exact DDA (reading Q13).

The oracle walk (oracle.c orc_trace_ray) is checked against things it does not
compute itself: hand-traced walks (tests/golden/dda_hand_traced.txt), the closed
form 1 + sum|floor(E) - floor(O)|, and an exact-rational brute-force membership
test over the bounding box (oracle/exact.py, Fractions, no event walk).
"""
import numpy as np
import pytest

import oracle
from oracle import exact
from nbt_inputs import random_segments_q16, tie_segments_q16, rand_map
from conftest import read_golden

Q = 65536   # Q16 walk coordinates (Q19)


def q16(xs):
    return [int(round(float(x) * Q)) for x in xs]


def all_state(code, n=8, policy=0, gain=(1.0, 0.12, 0.03)):
    return oracle.OracleMap(np.full((n, n, n), code, np.uint8), gain=gain, outside_policy=policy)


def closed_form(o, e):
    return 1 + sum(abs((int(e[k]) >> 16) - (int(o[k]) >> 16)) for k in range(3))


@pytest.mark.parametrize("row", read_golden("dda_hand_traced.txt"))
def test_hand_traced(row):
    name, o, e, seq = [s.strip() for s in row.split("|")]
    o, e = q16(o.split()), q16(e.split())
    want = [tuple(int(t) for t in v.split()) for v in seq.split(";")]
    m = all_state(1, n=4)  # all Free: nothing stops the walk
    ijk, codes, r = oracle.trace_ray(m, o, e)
    assert [tuple(v) for v in ijk] == want, name
    assert r.visits == len(want) == closed_form(o, e)


def test_closed_form_and_connectivity_random():
    """T2/T3/T7: 1 + sum|dfloor| voxels, consecutive voxels 6-adjacent, monotone per axis."""
    o_all, e_all = random_segments_q16(2000, -3.0, 11.0, seed=11)
    m = all_state(1)
    for o, e in zip(o_all, e_all):
        ijk, _, r = oracle.trace_ray(m, o, e, max_visits=256)
        assert r.visits == len(ijk) == closed_form(o, e)
        assert tuple(ijk[0]) == tuple(int(x) >> 16 for x in o)
        assert tuple(ijk[-1]) == tuple(int(x) >> 16 for x in e)
        steps = np.abs(np.diff(ijk, axis=0)).sum(1)
        assert (steps == 1).all()
        for k in range(3):
            dk = np.diff(ijk[:, k])
            assert (dk >= 0).all() or (dk <= 0).all()


def _brute_force_check(o, e, ijk):
    seq = [tuple(int(t) for t in v) for v in ijk]
    F = exact.floor_set(o, e)
    T = exact.touch_set(o, e)
    S = set(seq)
    assert len(S) == len(seq)                      # no voxel twice
    assert F <= S <= T
    if not exact.same_sign_ties(o, e):
        assert S == F
    # visiting order follows the entry parameter of the segment points
    ts = [exact.enter_param(o, e, v) for v in seq if v in F]
    assert all(a <= b for a, b in zip(ts, ts[1:]))


def test_brute_force_random_segments():
    """T8: F <= visited <= touched by exact slab tests; equality without same-sign ties."""
    o_all, e_all = random_segments_q16(300, 0.0, 8.0, seed=5)
    m = all_state(1)
    for o, e in zip(o_all, e_all):
        ijk, _, _ = oracle.trace_ray(m, o, e)
        _brute_force_check(o, e, ijk)


def test_brute_force_tie_segments():
    """T8 on segments whose endpoints lie on faces, edges and corners (exact ties)."""
    o_all, e_all = tie_segments_q16(300, 6, seed=9)
    m = all_state(1)
    n_ties = 0
    for o, e in zip(o_all, e_all):
        ijk, _, _ = oracle.trace_ray(m, o, e)
        _brute_force_check(o, e, ijk)
        n_ties += bool(exact.same_sign_ties(o, e))
    assert n_ties > 10   # the fixture really exercises ties


def test_early_stop_counts_hit_voxel():
    """T9: if the k-th visited voxel is the first Occupied one, exactly k voxels count,
    n_O = 1, and randomizing every later voxel changes nothing."""
    rng = np.random.default_rng(3)
    o_all, e_all = random_segments_q16(200, 0.2, 7.8, seed=21)
    for o, e in zip(o_all, e_all):
        free = all_state(1)
        ijk, _, _ = oracle.trace_ray(free, o, e)
        if len(ijk) < 2:
            continue
        k = int(rng.integers(1, len(ijk) + 1))
        codes = np.ones((8, 8, 8), np.uint8)
        for v in ijk[: k - 1]:
            codes[v[2], v[1], v[0]] = rng.integers(0, 2)
        hx, hy, hz = ijk[k - 1]
        codes[hz, hy, hx] = 2
        r1 = oracle.trace_ray(oracle.OracleMap(codes), o, e)[2]
        assert (r1.n_u + r1.n_f + r1.n_o, r1.n_o, r1.stop) == (k, 1, 1)
        later = {tuple(v) for v in ijk[k:]}
        codes2 = codes.copy()
        for v in later:
            codes2[v[2], v[1], v[0]] = rng.integers(0, 3)
        r2 = oracle.trace_ray(oracle.OracleMap(codes2), o, e)[2]
        assert (r2.n_u, r2.n_f, r2.n_o) == (r1.n_u, r1.n_f, r1.n_o)


def test_occupied_origin():
    """T10: Occupied origin voxel -> one voxel counted, g_R = g_O."""
    m = all_state(2, gain=(1.0, 0.12, 0.25))
    _, _, r = oracle.trace_ray(m, q16([3.5, 3.5, 3.5]), q16([7.5, 1.5, 2.5]))
    assert (r.n_u, r.n_f, r.n_o, r.stop) == (0, 0, 1, 1)
    assert r.g == 0.25


def test_monotone_free_to_unknown():
    """T12: flipping one traversed Free voxel to Unknown raises g_R by exactly 1 - g_F."""
    o, e = q16([0.3, 0.6, 0.9]), q16([7.7, 6.1, 5.3])
    base = np.ones((8, 8, 8), np.uint8)
    g0 = oracle.trace_ray(oracle.OracleMap(base, gain=(1.0, 0.25, 0.0)), o, e)[2].g
    ijk, _, _ = oracle.trace_ray(oracle.OracleMap(base), o, e)
    for v in ijk:
        c = base.copy(); c[v[2], v[1], v[0]] = 0
        g1 = oracle.trace_ray(oracle.OracleMap(c, gain=(1.0, 0.25, 0.0)), o, e)[2].g
        assert g1 - g0 == pytest.approx(0.75, abs=1e-12)


def test_outside_policy_and_tail():
    """Q14: outside the grid is Unknown (counted, no lookup) or clipped (not counted);
    once the walk leaves the grid it never re-enters."""
    codes = rand_map(8, seed=4)
    codes[codes == 2] = 1  # no early stop
    o_all, e_all = random_segments_q16(300, -4.0, 12.0, seed=8)
    for o, e in zip(o_all, e_all):
        mu = oracle.OracleMap(codes, outside_policy=0)
        mc = oracle.OracleMap(codes, outside_policy=1)
        ijk, cds, ru = oracle.trace_ray(mu, o, e)
        rc = oracle.trace_ray(mc, o, e)[2]
        inside = [(0 <= v).all() and (v < 8).all() for v in ijk]
        assert ru.lookups == rc.lookups == sum(inside)
        assert ru.n_u + ru.n_f == len(ijk)
        assert rc.n_u + rc.n_f == sum(inside)
        assert all(c == 255 for c, i in zip(cds, inside) if not i)
        # inside visits form one contiguous run
        idx = [i for i, b in enumerate(inside) if b]
        if idx:
            assert idx == list(range(idx[0], idx[-1] + 1))


def test_invalid_coordinates_rejected():
    m = all_state(1)
    with pytest.raises(oracle.OracleError):
        oracle.trace_ray(m, [0, 0, 0], [1 << 30, 0, 0])   # outside (-2^30, 2^30)
