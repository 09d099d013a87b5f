"""Pins of the oracle's IDW query (Eq. 4, T22), perspective sampler (Eq. 1, T20-T21),
Philox known answers and the S:69 state classification."""
import math

import numpy as np
import pytest

import oracle
from conftest import read_golden

SPEC = {}
for row in read_golden("spec_examples.txt"):
    k, *v = row.split()
    SPEC.setdefault(k, []).append([float(x) for x in v])


# ----------------------------------------------------------------- IDW (Eq. 4)

def test_idw_single_perspective():
    """single perspective gain 4.2, any query -> 4.2."""
    g = oracle.idw_query([([[1.0, 2.0, 3.0]], [4.2])], [[0.0, 0.0, 0.0], [5.0, -1.0, 2.0]])
    assert (g == SPEC["idw_single_4_2"][0][0]).all()


def test_idw_zero_distance():
    """S:227, Q23: query at a perspective origin -> that origin's gain."""
    xyz = [[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 2.0, 0.0]]
    g = oracle.idw_query([(xyz, [1.0, 3.0, 7.0])], [[1.0, 0.0, 0.0], [1.0 + 1e-12, 0.0, 0.0]])
    assert g[0] == 3.0 and g[1] == 3.0


def test_idw_pair_example():
    """gains {1, 3} at distances {1, 2}, p = 2 -> (1*1 + 3*0.25)/1.25 = 1.4."""
    g = oracle.idw_query([([[1.0, 0.0, 0.0], [-2.0, 0.0, 0.0]], [1.0, 3.0])], [[0.0, 0.0, 0.0]], power_p=2.0)
    assert g[0] == pytest.approx(SPEC["idw_pair_1_4"][0][0], rel=1e-15)


def test_idw_two_entries():
    """N_B = 2, entry values oldest 2, newest 4 -> 2*(1/2) + 4*1 = 5.0."""
    e_old = ([[0.0, 0.0, 0.0]], [2.0])
    e_new = ([[3.0, 0.0, 0.0]], [4.0])
    assert oracle.idw_query([e_old, e_new], [[1.0, 1.0, 1.0]])[0] == SPEC["gain_at_two_entries"][0][0]
    assert oracle.idw_query([e_old, e_new], [[1.0, 1.0, 1.0]], normalize=True)[0] == pytest.approx(5.0 / 1.5)


def test_idw_convex_and_harmonic():
    """S:258 (convex combination per entry) and S:261 (identical full buffer -> H_NB x value)."""
    rng = np.random.default_rng(0)
    xyz = rng.normal(size=(50, 3)); gain = rng.uniform(0, 5, 50)
    q = rng.normal(size=(100, 3)) * 2
    for p in (0.5, 1.0, 2.0, 3.0):
        v = oracle.idw_query([(xyz, gain)], q, power_p=p)
        assert (v >= gain.min() - 1e-12).all() and (v <= gain.max() + 1e-12).all()
    v = oracle.idw_query([(xyz, gain)], q)
    g10 = oracle.idw_query([(xyz, gain)] * 10, q)
    h10 = sum(1.0 / k for k in range(1, 11))
    assert np.allclose(g10, h10 * v, rtol=1e-13)


def test_idw_matches_direct_formula_p2():
    """Eq. 4 written out in numpy for p = 2 on a random buffer of 3 entries."""
    rng = np.random.default_rng(1)
    ents = [(rng.normal(size=(20, 3)), rng.uniform(0, 3, 20)) for _ in range(3)]
    q = rng.normal(size=(30, 3)) * 3
    got = oracle.idw_query(ents, q)
    want = np.zeros(30)
    for u, (x, g) in enumerate(ents):
        w = 1.0 / ((q[:, None, :] - x[None]) ** 2).sum(-1)
        want += (1.0 / (3 - u)) * (w * g).sum(1) / w.sum(1)
    assert np.allclose(got, want, rtol=1e-12)


def test_idw_empty_buffer():
    with pytest.raises(oracle.OracleError):
        oracle.idw_query([], [[0.0, 0.0, 0.0]])


# -------------------------------------------------------------- sampler (Eq. 1)

def test_philox_known_answers():
    for row in read_golden("philox_kat.txt"):
        v = [int(x, 16) for x in row.split()]
        assert oracle.philox4x32(v[:4], v[4:6]) == v[6:]


def test_forced_sample():
    """X = (1,0,0), X_R = 1, r_S = 1, PoI = 0 -> (1,0,0)."""
    p = oracle.eq1([0.0, 0.0, 0.0], 1.0, [1.0, 0.0, 0.0], 1.0)
    assert list(p) == SPEC["forced_sample"][0]
    p = oracle.eq1([1.0, 2.0, 3.0], 2.0, [0.0, -5.0, 0.0], 0.125)
    assert np.allclose(p, [1.0, 1.0, 3.0], atol=1e-15)


def test_sampler_radius_and_surface():
    """||p - PoI|| <= r_S; surface mode at r_S +- 1e-12; deterministic per seed."""
    poi = np.array([0.3, -1.0, 2.0])
    a = oracle.sample_perspectives(poi, 1.5, 20000, seed=42, mode=0)
    assert (np.linalg.norm(a - poi, axis=1) <= 1.5 * (1 + 1e-15)).all()
    s = oracle.sample_perspectives(poi, 1.5, 20000, seed=42, mode=1)
    assert np.abs(np.linalg.norm(s - poi, axis=1) - 1.5).max() < 1e-12
    assert np.array_equal(a, oracle.sample_perspectives(poi, 1.5, 20000, seed=42, mode=0))
    assert not np.array_equal(a, oracle.sample_perspectives(poi, 1.5, 20000, seed=43, mode=0))


def test_sampler_distribution():
    """T21: radial CDF (r/r_S)^3 (KS < 0.01), fraction inside r_S/2 = 0.125 +- 0.01,
    octant counts within 3 sigma, direction isotropy."""
    n = 100000
    p = oracle.sample_perspectives([0.0, 0.0, 0.0], 1.0, n, seed=7, mode=0)
    r = np.sort(np.linalg.norm(p, axis=1))
    ks = np.max(np.abs(np.arange(1, n + 1) / n - r ** 3))
    assert ks < 0.01
    assert abs((r <= 0.5).mean() - 0.125) < 0.01
    oct_ = (p[:, 0] > 0) * 4 + (p[:, 1] > 0) * 2 + (p[:, 2] > 0)
    cnt = np.bincount(oct_, minlength=8)
    sigma = math.sqrt(n * (1 / 8) * (7 / 8))
    assert (np.abs(cnt - n / 8) < 3 * sigma).all()
    u = p / np.linalg.norm(p, axis=1, keepdims=True)
    assert np.abs(u.mean(0)).max() < 0.02          # no preferred direction
    assert np.abs((u ** 2).mean(0) - 1 / 3).max() < 0.01


# --------------------------------------------------------- classification S:69

def test_classify_rules():
    """unstored/unobserved -> Unknown; P = 0.97 (t_occ 0.5) -> Occupied;
    an observed miss (P < 0.5) -> Free; observed P = 0.5 -> Occupied (rule order, Q16);
    with a band (t_occ 0.7, t_free 0.3) P = 0.5 -> Unknown."""
    p = np.array([0.97, 0.4, 0.5, 0.1, 0.97], np.float32)
    obs = np.array([1, 1, 1, 0, 0], np.uint8)
    assert list(oracle.classify(p, obs)) == [2, 1, 2, 0, 0]
    assert list(oracle.classify(p, obs, 0.7, 0.3)) == [2, 0, 0, 0, 0]


def test_idw_knn_hand_example_and_identities():
    """Optional k-nearest Eq. 4 (reading Q22): a hand example, k >= N_P equals the full
    sum bit for bit, k = 1 returns the nearest gain, equal distances go to the lower j."""
    P = np.array([[1.0, 0, 0], [0, 2.0, 0], [0, 0, 4.0]])
    g = np.array([1.0, 2.0, 3.0])
    x = np.zeros((1, 3))
    # k = 2: weights 1 and 1/4 -> (1*1 + 2/4) / (1 + 1/4) = 1.2
    v = oracle.idw_query_knn([(P, g)], x, 2)
    assert abs(v[0] - 1.2) < 1e-15
    rng = np.random.default_rng(3)
    Pr = rng.normal(size=(37, 3)); gr = rng.random(37); q = rng.normal(size=(20, 3)) * 2
    full = oracle.idw_query([(Pr, gr), (Pr[:11], gr[:11])], q)
    for k in (37, 50):
        assert np.array_equal(oracle.idw_query_knn([(Pr, gr), (Pr[:11], gr[:11])], q, k), full)
    # k = 1: the nearest perspective's gain (one term: g w / w)
    v1 = oracle.idw_query_knn([(Pr, gr)], q, 1)
    near = np.argmin(((q[:, None, :] - Pr[None]) ** 2).sum(-1), axis=1)
    np.testing.assert_allclose(v1, gr[near], rtol=1e-15)
    # ties: two perspectives at the same distance, k = 1 takes the lower index
    Pt = np.array([[0, 3.0, 0], [3.0, 0, 0], [0, 0, 9.0]]); gt = np.array([0.25, 0.75, 0.5])
    assert oracle.idw_query_knn([(Pt, gt)], x, 1)[0] == 0.25
    with pytest.raises(oracle.OracleError):
        oracle.idw_query_knn([(Pt, gt)], x, 0)
