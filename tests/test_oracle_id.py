"""Pins of the oracle's whole ID: frames, endpoints, scores, reduction
(SPEC worked examples)."""
import math

import numpy as np
import pytest

import oracle
from nbt_inputs import CONFIGS, FOV_H, FOV_V, rand_map, syn_map
from conftest import read_golden

Q = 65536
SPEC = {}
for row in read_golden("spec_examples.txt"):
    k, *v = row.split()
    SPEC.setdefault(k, []).append([float(x) for x in v])


def q16(v16):
    """The walk's segment ends are the Q16 lattice values themselves (
    reading Q19): no second rounding."""
    return np.asarray(v16, dtype=np.int64)


def one_ray_cam():
    return oracle.camera_from_fov(math.pi / 2, math.pi / 2, 1, 1)   # W = H = 1: the centre ray only


def test_spec_ray_gain_unknown_10():
    """fully unknown map, ray crossing exactly 10 voxels -> 10.0."""
    m = oracle.OracleMap(np.zeros((32, 32, 32), np.uint8))
    poi = [20.5, 16.5, 16.5]
    _, g, c = oracle.id_compute(m, poi, [[2.5, 16.5, 16.5]], one_ray_cam(), 9.0)
    assert g[0] == SPEC["ray_gain_unknown_10"][0][0]
    assert tuple(c[0]) == (10, 0, 0, 10)


def test_spec_first_voxel_occupied():
    """first voxel Occupied with P = 1 -> g_O = 1 - P = 0, then stop."""
    codes = np.zeros((32, 32, 32), np.uint8)
    codes[16, 16, 2] = 2
    m = oracle.OracleMap(codes, gain=(1.0, 0.12, 0.0))
    _, g, c = oracle.id_compute(m, [20.5, 16.5, 16.5], [[2.5, 16.5, 16.5]], one_ray_cam(), 9.0)
    assert g[0] == SPEC["ray_gain_first_occupied"][0][0]
    assert tuple(c[0]) == (0, 0, 1, 1)


def test_spec_distribution_one_ray_7():
    """N_P = 1, one ray over 7 unknown voxels -> 7.0 (along -y this time)."""
    m = oracle.OracleMap(np.zeros((16, 16, 16), np.uint8))
    _, g, _ = oracle.id_compute(m, [8.5, 1.5, 8.5], [[8.5, 12.5, 8.5]], one_ray_cam(), 6.0)
    assert g[0] == SPEC["distribution_one_ray_7"][0][0]


@pytest.mark.parametrize("key,d_cam,fov", [("d_h_2_pi2", 2.0, math.pi / 2), ("d_h_3_pi3", 3.0, math.pi / 3)])
def test_far_plane_half_extent(key, d_cam, fov):
    """T18: the corner rays sit at d_h = d_Cam tan(FoV_h/2) along right."""
    cam = oracle.camera_from_fov(fov, fov, 3, 3)
    m = oracle.OracleMap(np.zeros((4, 4, 4), np.uint8))
    f = oracle.frame(m, [0.0, 0.0, 0.0], [-5.0, 0.0, 0.0], cam, d_cam)
    d_h = np.linalg.norm(f["rc"]) / Q
    assert d_h == pytest.approx(SPEC[key][0][0], abs=2 ** -15)
    # corner pixel (i = W-1) of the lattice lands on the same border: 2 * Rh * (W-1)/2 = Rc
    assert np.abs(2 * f["rh"] - f["rc"]).max() <= 2


def test_frames_orthonormal_and_rays():
    """T17: unit, mutually orthogonal axes; centre ray ends at O + A; corners at O + A +- Rc +- Uc;
    fwd points at the PoI; up-hint fallback when fwd is parallel to z (Q4)."""
    rng = np.random.default_rng(1)
    m = oracle.OracleMap(np.zeros((8, 8, 8), np.uint8))
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 5, 3)
    cam.add_corners = 1
    poi = np.array([4.0, 4.0, 4.0])
    pts = list(poi + rng.normal(size=(200, 3)) * 3) + [poi + [0, 0, 2.5], poi - [0, 0, 1.0]]
    for p in pts:
        f = oracle.frame(m, poi, p, cam, 5.0)
        A = np.stack([f["fwd"], f["right"], f["up"]])
        assert np.abs(A @ A.T - np.eye(3)).max() < 1e-15 * 4
        d = poi - p
        assert np.allclose(f["fwd"], d / np.linalg.norm(d), atol=1e-15)
        o, e, _ = oracle.perspective_rays(m, poi, p, cam, 5.0, with_counts=False)
        assert (o == q16(f["o"])).all()
        centre = 1 * 5 + 2   # row kk = 1, column i = 2 of a 5 x 3 lattice
        assert (e[centre] == q16(f["o"] + f["a"])).all()
        for q, (sr, su) in enumerate([(-1, -1), (1, -1), (-1, 1), (1, 1)]):
            assert (e[15 + q] == q16(f["o"] + f["a"] + sr * f["rc"] + su * f["uc"])).all()
        # the lattice's 4 border pixels coincide with the corner rays to within rounding:
        # (W-1) Rh vs Rc, each rounded once per component -> at most (W-1)/2 + 1/2 units
        for q, idx in enumerate([0, 4, 10, 14]):
            assert np.abs(e[idx] - e[15 + q]).max() <= 3


def test_degenerate_perspective_rejected():
    """Q18: a perspective at the PoI has no orientation."""
    m = oracle.OracleMap(np.zeros((8, 8, 8), np.uint8))
    with pytest.raises(oracle.OracleError) as ei:
        oracle.id_compute(m, [4.0, 4.0, 4.0], [[1.0, 1.0, 1.0], [4.0, 4.0, 4.0]], one_ray_cam(), 3.0)
    assert ei.value.code == oracle.ERR_DEGENERATE


def test_closed_form_all_unknown():
    """T2 at perspective level: in an all-Unknown map g_P = mean_k (1 + sum_a |dfloor_a|)."""
    m = oracle.OracleMap(np.zeros((16, 16, 16), np.uint8))
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 9, 7)
    poi = [8.5, 8.5, 8.5]
    P = oracle.sample_perspectives(poi, 6.0, 12, seed=3)
    _, g, c = oracle.id_compute(m, poi, P, cam, 12.0)
    for j, p in enumerate(P):
        o, e, _ = oracle.perspective_rays(m, poi, p, cam, 12.0, with_counts=False)
        cnt = 1 + np.abs((e >> 16) - (o >> 16)[None, :]).sum(1)
        assert c[j, 0] == cnt.sum() and c[j, 1] == c[j, 2] == 0
        assert g[j] == cnt.sum() / cnt.size


def test_bounds_and_linearity():
    """T11 (0 <= g_P <= max ray count) and T13 (g_P linear in (g_U, g_F, g_O) with
    coefficients T_c / N_E)."""
    codes = rand_map(12, seed=2)
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 8, 6)
    poi = [6.5, 6.5, 6.5]
    P = oracle.sample_perspectives(poi, 5.0, 10, seed=4)
    gains = [(1.0, 0.12, 0.03), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0), (0.3, 0.7, 0.9)]
    res = [oracle.id_compute(oracle.OracleMap(codes, gain=gn), poi, P, cam, 10.0) for gn in gains]
    ne = 48
    for gn, (_, g, c) in zip(gains, res):
        assert (g >= 0).all()
        lin = (c[:, 0] * gn[0] + c[:, 1] * gn[1] + c[:, 2] * gn[2]) / ne
        assert np.allclose(g, lin, rtol=1e-14, atol=0)
    assert np.allclose(res[4][1], 0.3 * res[1][1] + 0.7 * res[2][1] + 0.9 * res[3][1], rtol=1e-13)
    # the per-state totals do not depend on the gain table
    for _, _, c in res[1:]:
        assert (c == res[0][2]).all()


def test_symmetry_all_unknown():
    """T14: perspectives mirrored through a voxel-centre PoI get identical totals in an
    all-Unknown map when no endpoint coordinate sits exactly on a voxel boundary."""
    m = oracle.OracleMap(np.zeros((40, 40, 40), np.uint8))
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 6, 5)
    poi = np.array([20.5, 20.5, 20.5])
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(40):
        d = rng.normal(size=3)
        d *= 7.0 / np.linalg.norm(d)
        p1, p2 = poi + d, poi - d
        _, e1, _ = oracle.perspective_rays(m, poi, p1, cam, 9.0, with_counts=False)
        _, e2, _ = oracle.perspective_rays(m, poi, p2, cam, 9.0, with_counts=False)
        if ((e1 & 0xFFF) == 0).any() or ((e2 & 0xFFF) == 0).any():
            continue
        _, _, c = oracle.id_compute(m, poi, [p1, p2], cam, 9.0)
        assert (c[0, :3] == c[1, :3]).all()
        checked += 1
    assert checked > 30


def test_empty_fov_gives_zero():
    """T15: all-Free map with g_F = 0 -> 0; occupied origin voxels with g_O = 0 -> 0."""
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 7, 5)
    poi = [6.5, 6.5, 6.5]
    P = oracle.sample_perspectives(poi, 4.0, 8, seed=1)
    free = oracle.OracleMap(np.ones((13, 13, 13), np.uint8), gain=(1.0, 0.0, 0.03), outside_policy=1)
    assert (oracle.id_compute(free, poi, P, cam, 20.0)[1] == 0).all()
    occ = oracle.OracleMap(np.full((13, 13, 13), 2, np.uint8), gain=(1.0, 0.12, 0.0))
    _, g, c = oracle.id_compute(occ, poi, P, cam, 20.0)
    assert (g == 0).all() and (c[:, 2] == 35).all() and (c[:, :2] == 0).all()


def test_permutation_and_determinism():
    """T16/T23: per-perspective results are independent of order, thread count and run."""
    codes = rand_map(16, seed=12)
    m = oracle.OracleMap(codes)
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 8, 6)
    poi = [8.5, 8.5, 8.5]
    P = oracle.sample_perspectives(poi, 6.0, 24, seed=5)
    a = oracle.id_compute(m, poi, P, cam, 12.0, nthreads=1)
    b = oracle.id_compute(m, poi, P, cam, 12.0, nthreads=4)
    perm = np.random.default_rng(0).permutation(24)
    c = oracle.id_compute(m, poi, P[perm], cam, 12.0, nthreads=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(a[1][perm], c[1]) and np.array_equal(a[2][perm], c[2])


def test_grid_scaling_counts():
    """s_G lattice (Q6-Q9): dedup example and the N_E of BASELINE.md 'Derived'."""
    cam = oracle.camera_from_grid_scaling(math.pi / 2, math.pi / 2, 2.0, 0.01, 100.0)
    assert oracle.num_rays(cam) == SPEC["grid_count_dedup"][0][0]
    for s_g, ne in SPEC["grid_count_sg"]:
        cam = oracle.camera_from_grid_scaling(FOV_H, FOV_V, 3.86, 0.01, s_g)
        assert oracle.num_rays(cam) == ne


def test_grid_scaling_spacing():
    """Lattice rays are s_G voxels apart on the far plane and the corner rays reach d_h, d_v."""
    cam = oracle.camera_from_grid_scaling(FOV_H, FOV_V, 0.5, 0.01, 10.0)
    m = oracle.OracleMap(np.zeros((4, 4, 4), np.uint8), voxel_size=0.01)
    poi = [0.0, 0.0, 0.0]
    p = [-0.6, 0.1, 0.05]
    f = oracle.frame(m, poi, p, cam, 0.5)
    assert np.linalg.norm(2 * f["rh"]) / Q == pytest.approx(10.0, abs=1e-4)
    _, e, _ = oracle.perspective_rays(m, poi, p, cam, 0.5, with_counts=False)
    nl = cam.width * cam.height
    centre = e[(cam.height // 2) * cam.width + cam.width // 2]
    off = (e[nl + 3] - centre) / 65536.0
    assert np.linalg.norm(off) == pytest.approx(50 * math.hypot(math.tan(FOV_H / 2), math.tan(FOV_V / 2)), rel=1e-5)


def test_soft_trend_closer_scores_lower():
    """T24: on the synthetic scene, perspectives nearer the object score lower
    (positive rank correlation of distance to the PoI vs g_P)."""
    cfg = CONFIGS["A"]
    m = oracle.OracleMap(syn_map(cfg.n, cfg.r_o, cfg.map_seed), voxel_size=cfg.voxel_size)
    cam = oracle.camera_from_fov(FOV_H, FOV_V, 16, 12)
    P = oracle.sample_perspectives(cfg.poi, 28.0, 64, seed=2, mode=0)
    _, g, _ = oracle.id_compute(m, cfg.poi, P, cam, cfg.range_, nthreads=4)
    d = np.linalg.norm(P - cfg.poi, axis=1)
    rd, rg = np.argsort(np.argsort(d)), np.argsort(np.argsort(g))
    rho = np.corrcoef(rd, rg)[0, 1]
    assert rho > 0.1   # positive; measured 0.25 here
