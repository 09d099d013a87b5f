"""Pins of the oracle's per-voxel-probability mode (Eq. 2 with each voxel's
P(v); reading Q32: P quantised to level/63)."""
import math

import numpy as np
import pytest

import oracle
from nbt_inputs import FOV_H, FOV_V, rand_map

Q = 65536   # Q16 walk coordinates (Q19)


def one_ray_cam():
    return oracle.camera_from_fov(math.pi / 2, math.pi / 2, 1, 1)


def test_quantize_prob_examples():
    """S:69 states with level = rne(63 P): 0.5 -> 32 (31.5, half to even), 0.97 -> 61,
    0.12 -> 8, 1.0 -> 63, unobserved -> (Unknown, 0); with a band (0.7, 0.3) P = 0.5 -> Unknown."""
    p = np.array([0.5, 0.97, 0.12, 1.0, 0.3], np.float32)
    obs = np.array([1, 1, 1, 1, 0], np.uint8)
    codes, levels = oracle.quantize_prob(p, obs)
    assert list(codes) == [2, 2, 1, 2, 0]
    assert list(levels) == [32, 61, 8, 63, 0]
    codes, _ = oracle.quantize_prob(p, obs, 0.7, 0.3)
    assert list(codes) == [0, 2, 1, 2, 0]


def test_hand_ray_eq2():
    """One ray through Free voxels with P = 0, 10/63, 20/63, 30/63, 1 and then an Occupied voxel
    with P = 60/63: g_R = (0 + 10 + 20 + 30 + 63 + (63 - 60)) / 63 and the walk stops there."""
    codes = np.zeros((3, 3, 12), np.uint8)
    levels = np.zeros_like(codes)
    codes[1, 1, 1:6] = 1
    levels[1, 1, 1:6] = [0, 10, 20, 30, 63]
    codes[1, 1, 6] = 2
    levels[1, 1, 6] = 60
    m = oracle.OracleMap(codes, levels=levels)
    _, g, c, tg = oracle.id_compute(m, [11.5, 1.5, 1.5], [[1.5, 1.5, 1.5]], one_ray_cam(), 9.0, with_tg=True)
    assert tg[0] == 0 + 10 + 20 + 30 + 63 + 3
    assert g[0] == pytest.approx(126 / 63, rel=1e-15)
    assert tuple(c[0]) == (0, 5, 1, 6)


def test_uniform_levels_equal_per_state_mode():
    """With every Free voxel at level 8 and every Occupied at level 61, the exact Eq. 2 equals
    the per-state constants (1, 8/63, 2/63): same totals, g_P within 1e-13."""
    codes = rand_map(16, 0.3, 0.65, 0.05, seed=3)
    levels = np.where(codes == 1, 8, np.where(codes == 2, 61, 0)).astype(np.uint8)
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 9, 7)
    poi = [8.5, 8.5, 8.5]
    P = oracle.sample_perspectives(poi, 6.0, 20, seed=1)
    a = oracle.id_compute(oracle.OracleMap(codes, levels=levels), poi, P, cam, 14.0)
    b = oracle.id_compute(oracle.OracleMap(codes, gain=(1.0, 8 / 63, 2 / 63)), poi, P, cam, 14.0)
    assert np.array_equal(a[2], b[2])
    assert np.allclose(a[1], b[1], rtol=1e-13)


def test_monotone_in_probability():
    """Eq. 2: raising P of a traversed Free voxel raises g_R by the same amount; raising P of the
    Occupied voxel that stops the ray lowers g_R by it."""
    codes = np.ones((3, 3, 10), np.uint8)
    codes[1, 1, 8] = 2
    lv = np.full_like(codes, 20)
    cam = one_ray_cam()
    base = oracle.id_compute(oracle.OracleMap(codes, levels=lv), [9.5, 1.5, 1.5], [[0.5, 1.5, 1.5]], cam, 9.0,
                             with_tg=True)[3][0]
    lv2 = lv.copy(); lv2[1, 1, 3] = 33
    up = oracle.id_compute(oracle.OracleMap(codes, levels=lv2), [9.5, 1.5, 1.5], [[0.5, 1.5, 1.5]], cam, 9.0,
                           with_tg=True)[3][0]
    lv3 = lv.copy(); lv3[1, 1, 8] = 33
    down = oracle.id_compute(oracle.OracleMap(codes, levels=lv3), [9.5, 1.5, 1.5], [[0.5, 1.5, 1.5]], cam, 9.0,
                             with_tg=True)[3][0]
    assert up - base == 13 and base - down == 13


def test_map_update_hand_example():
    """Row a2 / Q30 on a hand-worked example: deltas apply in array order, so a voxel named
    twice ends with the later code; untouched voxels keep theirs; out-of-grid or code >= 3
    deltas are rejected."""
    codes = np.zeros((2, 3, 4), np.uint8)            # [z, y, x]
    m = oracle.OracleMap(codes)
    oracle.map_update(m, np.array([[1, 2, 0], [3, 0, 1], [1, 2, 0]], np.int32), np.array([1, 2, 2], np.uint8))
    want = np.zeros((2, 3, 4), np.uint8)
    want[0, 2, 1] = 2                                 # (x=1, y=2, z=0): 1 then 2
    want[1, 0, 3] = 2                                 # (x=3, y=0, z=1)
    assert np.array_equal(m.codes, want)
    with pytest.raises(oracle.OracleError):
        oracle.map_update(m, np.array([[4, 0, 0]], np.int32), np.array([1], np.uint8))
    with pytest.raises(oracle.OracleError):
        oracle.map_update(m, np.array([[0, 0, 0]], np.int32), np.array([3], np.uint8))
