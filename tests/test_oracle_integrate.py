"""Pins for the map-integration oracle: voxel filter, log-odds
integration with free-space carving, log-odds classification.

Citations: S:n = SPEC.md line n (the paper defers occupancy mapping to its framework,
P:84); Qn = DESIGN.md readings.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import exact
import nbt_inputs as I

LH = np.float32(math.log(0.7 / 0.3))
LM = np.float32(math.log(0.4 / 0.6))
LMIN = np.float32(math.log(0.12 / 0.88))
LMAX = np.float32(math.log(0.97 / 0.03))


def sig(x):
    return 1.0 / (1.0 + math.exp(-float(x)))


# ------------------------------------------------------------------ voxel filter

def test_filter_cube_corners_give_centre():
    """8 corners of a cube of edge 0.5, leaf 2.0 -> 1 point at the cube centre."""
    c = np.array([0.25, 0.25, 0.25])
    pts = np.array([[c[0] + dx, c[1] + dy, c[2] + dz] for dx in (0, 0.5) for dy in (0, 0.5) for dz in (0, 0.5)])
    out, cnt = oracle.voxel_filter(pts, 2.0)
    assert out.shape == (1, 3) and cnt.tolist() == [8]
    assert np.array_equal(out[0], c + 0.25)


def test_filter_single_point_identity():
    """one point, any leaf -> the same point (bit for bit)."""
    p = np.array([[0.123456789, -7.5, 3.25]])
    for leaf in (0.01, 1.0, 100.0):
        out, cnt = oracle.voxel_filter(p, leaf)
        assert np.array_equal(out, p) and cnt.tolist() == [1]


def test_filter_random_matches_bucketing():
    """1000 random points in the unit box, leaf 0.1 -> one point per distinct cell,
    each the mean of its cell; cells in ascending (iz, iy, ix) order (Q33)."""
    rng = np.random.default_rng(5)
    pts = rng.random((1000, 3))
    out, cnt = oracle.voxel_filter(pts, 0.1)
    cells = np.floor(pts / 0.1).astype(np.int64)
    uniq = {tuple(c) for c in cells}
    assert len(out) == len(uniq) and cnt.sum() == 1000
    keys = [(c[2], c[1], c[0]) for c in sorted(uniq, key=lambda c: (c[2], c[1], c[0]))]
    for j, (kz, ky, kx) in enumerate(keys):
        sel = (cells[:, 0] == kx) & (cells[:, 1] == ky) & (cells[:, 2] == kz)
        assert cnt[j] == sel.sum()
        np.testing.assert_allclose(out[j], pts[sel].mean(axis=0), rtol=0, atol=1e-15)
        assert np.array_equal(np.floor(out[j] / 0.1).astype(np.int64), [kx, ky, kz])


def test_filter_edge_cases():
    out, cnt = oracle.voxel_filter(np.zeros((0, 3)), 0.5)
    assert out.shape == (0, 3)
    with pytest.raises(oracle.OracleError):
        oracle.voxel_filter(np.array([[0.0, np.nan, 0.0]]), 0.5)
    with pytest.raises(oracle.OracleError):
        oracle.voxel_filter(np.array([[0.0, 0.0, 0.0]]), 0.0)
    # cell-index range (Q33): |cell| <= 32766 accepted, 32767 rejected
    out, cnt = oracle.voxel_filter(np.array([[32766.5, -32765.5, 0.0]]), 1.0)
    assert cnt.tolist() == [1]
    for bad in ([32767.5, 0.0, 0.0], [0.0, -32766.5, 0.0]):
        with pytest.raises(oracle.OracleError):
            oracle.voxel_filter(np.array([bad]), 1.0)
    # negative coordinates floor downwards
    out, cnt = oracle.voxel_filter(np.array([[-0.05, 0.0, 0.0], [-0.01, 0.0, 0.0], [0.01, 0.0, 0.0]]), 0.1)
    assert cnt.tolist() == [2, 1]


# ------------------------------------------------------------------ integration

def _grid(n=30):
    return oracle.new_logodds((n, n, n))


def test_single_point_hit_and_misses():
    """empty map, one point 1 m ahead, s_Vox = 0.1 -> the endpoint voxel has P = 0.7
    after one hit; the voxels before it one miss each (P = 0.4)."""
    L = _grid()
    touched, nr = oracle.integrate(L, 0.1, (0, 0, 0), (0.55, 1.55, 1.55), [[1.55, 1.55, 1.55]])
    assert nr == 1
    row = L[15, 15]
    assert row[15] == LH and abs(sig(row[15]) - 0.7) < 1e-6
    assert np.all(row[5:15] == LM) and abs(sig(LM) - 0.4) < 1e-6
    assert np.isnan(row[:5]).all() and np.isnan(row[16:]).all()
    assert int((touched > 0).sum()) == 11 and touched[15, 15, 15] == 3
    assert np.isnan(L).sum() == L.size - 11


def test_zero_points_unchanged():
    """zero points -> map unchanged."""
    L = _grid()
    L[3, 4, 5] = 1.25
    before = L.copy()
    touched, nr = oracle.integrate(L, 0.1, (0, 0, 0), (0.55, 1.55, 1.55), np.zeros((0, 3)))
    assert nr == 0 and not touched.any()
    assert np.array_equal(L, before, equal_nan=True)


def test_fifty_hits_clamp_at_pmax():
    """the same point 50 times -> endpoint P = P_max; the carved voxels P_min."""
    L = _grid()
    for _ in range(50):
        oracle.integrate(L, 0.1, (0, 0, 0), (0.55, 1.55, 1.55), [[1.55, 1.55, 1.55]])
    assert L[15, 15, 15] == LMAX and abs(sig(LMAX) - 0.97) < 1e-6
    assert np.all(L[15, 15, 5:15] == LMIN) and abs(sig(LMIN) - 0.12) < 1e-6
    # and the hand-computed approach to the clamp: k hits = min(k * L_hit, L_max) in float
    L2 = _grid()
    acc = np.float32(0.0)
    for k in range(1, 6):
        oracle.integrate(L2, 0.1, (0, 0, 0), (0.55, 1.55, 1.55), [[1.55, 1.55, 1.55]])
        acc = min(np.float32(acc + LH), LMAX)
        assert L2[15, 15, 15] == acc


def test_miss_is_free_hit_is_occupied():
    """observed once as a miss -> Free; a hit -> Occupied; unobserved -> Unknown."""
    L = _grid()
    oracle.integrate(L, 0.1, (0, 0, 0), (0.55, 1.55, 1.55), [[1.55, 1.55, 1.55]])
    codes, levels = oracle.occ_classify(L)
    assert codes[15, 15, 15] == 2 and np.all(codes[15, 15, 5:15] == 1) and codes[0, 0, 0] == 0
    assert levels[15, 15, 15] == round(63 * 0.7) and levels[15, 15, 7] == round(63 * 0.4) and levels[0, 0, 0] == 0


def test_hit_wins_over_miss_in_one_cloud():
    """Q35: a voxel that ends one ray and is crossed by another gets the hit only."""
    L = _grid()
    o = (0.05, 0.55, 0.55)
    touched, _ = oracle.integrate(L, 0.1, (0, 0, 0), o, [[0.55, 0.55, 0.55], [1.55, 0.55, 0.55]])
    row = L[5, 5]
    assert row[5] == LH and row[15] == LH
    assert np.all(row[0:5] == LM) and np.all(row[6:15] == LM)
    # order of the rays does not matter (set semantics)
    L2 = _grid()
    oracle.integrate(L2, 0.1, (0, 0, 0), o, [[1.55, 0.55, 0.55], [0.55, 0.55, 0.55]])
    assert np.array_equal(L, L2, equal_nan=True)


def test_range_truncation_carves_only():
    """S:61 errors: a point beyond max_range is cut at the range and only carves."""
    L = _grid(40)
    o = np.array([0.55, 2.05, 2.05])
    p = np.array([3.55, 2.05, 2.05])                # 3 m away
    touched, _ = oracle.integrate(L, 0.1, (0, 0, 0), o, [p], max_range=1.0)
    assert not (touched == 3).any()
    xs = np.argwhere(touched > 0)[:, 2]
    assert xs.min() == 5 and xs.max() == 15          # cut end 1.55 m -> voxel 15, carved
    assert np.all(L[20, 20, 5:16] == LM) and np.isnan(L[20, 20, 16:]).all()
    # within range: a hit
    L2 = _grid(40)
    touched, _ = oracle.integrate(L2, 0.1, (0, 0, 0), o, [p], max_range=5.0)
    assert touched[20, 20, 35] == 3


def test_touch_set_is_exact_segment_voxel_set():
    """The voxels one ray marks are exactly {floor(P(t)) : t in [0,1]} inside the grid
    (exact rational brute force), for endpoints on the Q16 lattice (s = 1, origin 0)."""
    rng = np.random.default_rng(17)
    n = 12
    for _ in range(60):
        o16 = rng.integers(-2 * 65536, (n + 2) * 65536, 3)
        e16 = rng.integers(-2 * 65536, (n + 2) * 65536, 3)
        L = oracle.new_logodds((n, n, n))
        touched, _ = oracle.integrate(L, 1.0, (0, 0, 0), o16 / 65536.0, [e16 / 65536.0], max_range=0.0)
        want = {v for v in exact.floor_set(o16, e16) if all(0 <= c < n for c in v)}
        got = {(int(x), int(y), int(z)) for z, y, x in np.argwhere(touched > 0)}
        assert got == want
        end = tuple(int(c) // 65536 for c in e16)
        if all(0 <= c < n for c in end):
            assert touched[end[2], end[1], end[0]] == 3
            assert int((touched == 3).sum()) == 1
        else:
            assert not (touched == 3).any()


def test_no_voxel_beyond_endpoint_is_carved():
    """no voxel beyond the first endpoint along a ray is marked free by that ray."""
    rng = np.random.default_rng(3)
    o = np.array([1.5, 1.5, 1.5])
    for _ in range(30):
        p = o + rng.uniform(-1.2, 1.2, 3)
        L = _grid()
        touched, _ = oracle.integrate(L, 0.1, (0, 0, 0), o, [p])
        d = p - o
        for z, y, x in np.argwhere(touched > 0):
            c = (np.array([x, y, z]) + 0.5) * 0.1
            t = float((c - o) @ d) / float(d @ d)
            assert t <= 1.0 + 0.1 * math.sqrt(3) / math.sqrt(float(d @ d))


def test_integrate_order_independent_and_filter_composes():
    """Q35 per-cloud set update: any permutation of a cloud gives the same store bit for
    bit; integrating with leaf > 0 equals integrating the filtered cloud with leaf 0."""
    cf = I.CLOUD_CONFIGS["F0"]
    pts = cf.cloud(0)
    L1 = oracle.new_logodds((cf.n,) * 3)
    oracle.integrate(L1, cf.voxel_size, (0, 0, 0), cf.sensor(0), pts, leaf=cf.leaf, max_range=cf.max_range)
    L2 = oracle.new_logodds((cf.n,) * 3)
    filt, _ = oracle.voxel_filter(pts, cf.leaf)
    perm = np.random.default_rng(0).permutation(len(filt))
    oracle.integrate(L2, cf.voxel_size, (0, 0, 0), cf.sensor(0), filt[perm], leaf=0.0, max_range=cf.max_range)
    assert np.array_equal(L1.view(np.uint32), L2.view(np.uint32))


def test_rejects_bad_input():
    L = _grid()
    with pytest.raises(oracle.OracleError):
        oracle.integrate(L, 0.1, (0, 0, 0), (0.5, 0.5, 0.5), [[np.inf, 0, 0]])
    with pytest.raises(oracle.OracleError):
        oracle.integrate(L, 0.1, (0, 0, 0), (0.5, 0.5, 0.5), [[1, 1, 1]], p_hit=1.0)


# ------------------------------------------------------------------ classification

def test_levels_are_round_63_sigmoid_away_from_boundaries():
    rng = np.random.default_rng(9)
    L = rng.uniform(-6, 6, 20000).astype(np.float32)
    codes, levels = oracle.occ_classify(L)
    for l, lv in zip(L[:4000], levels[:4000]):
        x = 63.0 * sig(l)
        if abs(x - math.floor(x) - 0.5) > 1e-4:
            assert lv == math.floor(x + 0.5)
    assert np.all(np.diff(levels[np.argsort(L)].astype(int)) >= 0)
    c, lv = oracle.occ_classify(np.array([LMAX, LMIN, np.nan, 0.0, -1e-30], np.float32))
    assert lv.tolist() == [61, 8, 0, 32, 31]
    assert c.tolist() == [2, 1, 0, 2, 1]           # t_occ = t_free = 0.5: P = 0.5 is Occupied


def test_band_thresholds():
    """with t_free < P < t_occ an observed voxel stays Unknown."""
    L = np.array([0.0, math.log(0.8 / 0.2), math.log(0.2 / 0.8), np.nan], np.float32)
    c, _ = oracle.occ_classify(L, t_occ=0.7, t_free=0.3)
    assert c.tolist() == [0, 2, 1, 0]
