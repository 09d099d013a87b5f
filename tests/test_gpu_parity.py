"""CUDA path (libnbt via its C ABI) vs the CPU oracle, element by element on the same seeded
inputs.  Integer results (visited voxel sequences, per-state totals, lookups, map codes)
must be bit-exact; g_P must be bit-exact too (same canonical fp64 expression, Q26); the
sampler and IDW (different transcendental / summation order) within 1e-12 relative."""
import math
import os

import numpy as np
import pytest

import oracle
from nbt_inputs import CONFIGS, FOV_H, FOV_V, Q16, rand_map, random_segments_q16, tie_segments_q16, syn_map

pytestmark = pytest.mark.gpu

NTHREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def nbt():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2503_22588_b200 import _build
    _build.build()
    import paper_2503_22588_b200 as mod
    return mod


@pytest.fixture(scope="module")
def ctx(nbt):
    return nbt.Ctx(0)


def make_map(nbt, ctx, codes, voxel_size=1.0, origin=(0.0, 0.0, 0.0), gain=None, policy=0, layout="linear",
             bits=2):
    """Device map (store layout and bits per voxel chosen through the descriptor) + oracle map."""
    nz, ny, nx = codes.shape
    m = nbt.Map(ctx, nbt.map_desc(nx, ny, nz, voxel_size, origin, gain, policy, layout=layout, state_bits=bits))
    m.upload(codes)
    om = oracle.OracleMap(codes, voxel_size=voxel_size, origin=origin,
                          gain=gain if gain is not None else (1.0, 0.12, 0.03), outside_policy=policy)
    return m, om


def run_both(nbt, ctx, m, om, poi, persp, w, h, range_, corners=False, grid=None):
    if grid is None:
        cam = nbt.camera_from_fov(FOV_H, FOV_V, w, h)
        ocam = oracle.camera_from_fov(FOV_H, FOV_V, w, h)
        cam.add_corners = ocam.add_corners = int(corners)
    else:
        cam = nbt.camera_from_grid_scaling(*grid)
        ocam = oracle.camera_from_grid_scaling(*grid)
    cloud = nbt.id_compute(ctx, m, poi, persp, cam, range_)
    _, g, c = oracle.id_compute(om, poi, persp, ocam, range_, nthreads=NTHREADS)
    return cloud, g, c


def assert_cloud_equal(cloud, persp, g, c):
    assert np.array_equal(np.asarray(cloud.xyz), np.asarray(persp))
    assert np.array_equal(cloud.counts.astype(np.int64), c)
    assert np.array_equal(cloud.gain, g)          # same canonical expression -> bit-exact


# ------------------------------------------------------------------ map store

def test_map_roundtrip_ragged(nbt, ctx):
    codes = rand_map(0, seed=3, shape=(11, 23, 37))
    m, _ = make_map(nbt, ctx, codes)
    assert np.array_equal(m.download(), codes)
    fresh = nbt.Map(ctx, nbt.map_desc(5, 6, 7, 1.0))
    assert (fresh.download() == 0).all()          # created all Unknown


def test_map_upload_rejects_bad_codes(nbt, ctx):
    codes = rand_map(8, seed=1)
    m, _ = make_map(nbt, ctx, codes)
    bad = codes.copy(); bad[3, 4, 5] = 3
    with pytest.raises(nbt.NbtError):
        m.upload(bad)
    assert np.array_equal(m.download(), codes)


def test_map_upload_prob_matches_classify(nbt, ctx):
    rng = np.random.default_rng(0)
    p = rng.uniform(0, 1, (9, 10, 11)).astype(np.float32)
    p[0, 0, :4] = [0.5, 0.3, 0.7, 0.12]
    obs = (rng.uniform(size=p.shape) < 0.8).astype(np.uint8)
    m = nbt.Map(ctx, nbt.map_desc(11, 10, 9, 1.0))
    for t_occ, t_free in [(0.5, 0.5), (0.7, 0.3)]:
        m.upload_prob(p, obs, t_occ, t_free)
        want = oracle.classify(p, obs, t_occ, t_free).reshape(p.shape)
        assert np.array_equal(m.download(), want)


def _apply_in_order(codes, ijk, vals):
    out = codes.copy()
    for (x, y, z), v in zip(ijk, vals):
        out[z, y, x] = v
    return out


@pytest.mark.parametrize("n", [5000, 20000])
@pytest.mark.parametrize("form", ["winner", "sort"])
@pytest.mark.parametrize("on_device", [False, True])
def test_map_update_last_wins(nbt, ctx, on_device, form, n):
    """Duplicated voxels resolve to the last delta (Q30), in both update forms (the
    winner array -- one single-block launch up to 8192 deltas, two grid-wide passes above --
    and the radix sort used when the array is absent), over repeated updates."""
    import torch
    ctx.set_option(nbt.OPT_DELTA_SORT, int(form == "sort"))
    codes = rand_map(0, seed=5, shape=(13, 17, 19))
    m, _ = make_map(nbt, ctx, codes)
    rng = np.random.default_rng(2)
    for rep in range(3):
        ijk = np.stack([rng.integers(0, 19, n), rng.integers(0, 17, n), rng.integers(0, 13, n)], 1).astype(np.int32)
        ijk[n // 2:] = ijk[: n - n // 2]                  # many duplicates
        vals = rng.integers(0, 3, n).astype(np.uint8)
        if on_device:
            m.update(torch.from_numpy(ijk).cuda(), torch.from_numpy(vals).cuda())
        else:
            m.update(ijk, vals)
        ctx.sync()
        codes = _apply_in_order(codes, ijk, vals)
        assert np.array_equal(m.download(), codes)
    ctx.set_option(nbt.OPT_DELTA_SORT, 0)


def test_map_update_validation(nbt, ctx):
    import torch
    m, _ = make_map(nbt, ctx, rand_map(6, seed=1))
    with pytest.raises(nbt.NbtError):
        m.update(np.array([[6, 0, 0]], np.int32), np.array([1], np.uint8))
    with pytest.raises(nbt.NbtError):
        m.update(np.array([[0, 0, 0]], np.int32), np.array([3], np.uint8))
    # device input: invalid entries are skipped and reported by the next sync
    before = m.download()
    m.update(torch.tensor([[0, 0, 0], [-1, 2, 2]], dtype=torch.int32, device="cuda"),
             torch.tensor([2, 1], dtype=torch.uint8, device="cuda"))
    with pytest.raises(nbt.NbtError):
        ctx.sync()
    after = before.copy(); after[0, 0, 0] = 2
    assert np.array_equal(m.download(), after)
    ctx.sync()                                        # error cleared


# ------------------------------------------------------------ per-ray walks

def _compare_walks(nbt, ctx, m, om, o, e, max_visits=256):
    ijk, cd, ln, cnt = nbt.debug_trace(ctx, m, o, e, max_visits)
    for r in range(len(o)):
        w_ijk, w_cd, w = oracle.trace_ray(om, o[r], e[r], max_visits)
        k = min(ln[r], max_visits)
        assert ln[r] == w.visits
        assert np.array_equal(ijk[r, :k], w_ijk[:k]), r
        assert np.array_equal(cd[r, :k], w_cd[:k]), r
        assert tuple(cnt[r]) == (w.n_u, w.n_f, w.n_o, w.lookups), r


@pytest.mark.parametrize("policy", [0, 1])
def test_walks_random_segments(nbt, ctx, policy):
    """Every visited voxel of 3000 random rays, inside, leaving and outside the grid."""
    codes = rand_map(12, 0.3, 0.68, 0.02, seed=7)
    m, om = make_map(nbt, ctx, codes, policy=policy)
    o, e = random_segments_q16(3000, -5.0, 17.0, seed=policy + 1)
    _compare_walks(nbt, ctx, m, om, o, e)


def test_walks_ties(nbt, ctx):
    """Endpoints on faces, edges and corners (exact ties of the DDA)."""
    codes = rand_map(8, 0.4, 0.6, 0.0, seed=2)
    m, om = make_map(nbt, ctx, codes)
    o, e = tie_segments_q16(4000, 9, seed=4)
    o -= Q16
    _compare_walks(nbt, ctx, m, om, o, e)


def test_walks_hand_traced(nbt, ctx):
    from conftest import read_golden
    m, om = make_map(nbt, ctx, np.ones((4, 4, 4), np.uint8))
    for row in read_golden("dda_hand_traced.txt"):
        _, o, e, seq = [s.strip() for s in row.split("|")]
        o = [int(round(float(v) * Q16)) for v in o.split()]
        e = [int(round(float(v) * Q16)) for v in e.split()]
        want = [tuple(int(t) for t in v.split()) for v in seq.split(";")]
        ijk, _, ln, _ = nbt.debug_trace(ctx, m, [o], [e], 16)
        assert [tuple(v) for v in ijk[0, :ln[0]]] == want


def test_walks_long_rays(nbt, ctx):
    """Long walks (1000+ voxels) through a sparse map: no drift of the decision terms."""
    codes = rand_map(64, 0.5, 0.5, 0.0, seed=9)
    m, om = make_map(nbt, ctx, codes)
    o, e = random_segments_q16(200, -30.0, 94.0, seed=12)
    _compare_walks(nbt, ctx, m, om, o, e, max_visits=400)


# ------------------------------------------- per-ray parity of the production trace kernel

def _per_ray_check(nbt, ctx, m, om, poi, P, cam, ocam, range_):
    rays = nbt.debug_id_rays(ctx, m, poi, P, cam, range_)
    cloud = nbt.id_compute(ctx, m, poi, P, cam, range_)
    for j in range(len(P)):
        _, _, want = oracle.perspective_rays(om, poi, P[j], ocam, range_)
        assert np.array_equal(rays[j].astype(np.int64), want), j
    # the recorded rays sum to the production kernel's per-perspective totals
    assert np.array_equal(rays[:, :, :4].sum(1, dtype=np.int64), cloud.counts.astype(np.int64))


def test_production_trace_per_ray_config_a(nbt, ctx):
    """All 12,288 rays of config A through the production k_id_trace code (batched walk,
    ffs/popc stop masks, refill queue) in its record instance: every ray's (n_U, n_F, n_O,
    lookups, stop) equals the oracle's (P:213 early stop, Q11-Q14), bit for bit."""
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    _per_ray_check(nbt, ctx, m, om, cfg.poi, P, cam, ocam, cfg.range_)


def test_production_trace_per_ray_config_b_subset(nbt, ctx):
    """Config B's map and camera, 6 of its perspectives (18,432 rays): per-ray parity of the
    production trace kernel."""
    cfg = CONFIGS["B"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)[::85][:6]
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    _per_ray_check(nbt, ctx, m, om, cfg.poi, P, cam, ocam, cfg.range_)


@pytest.mark.parametrize("layout,bits,policy", [("linear", 2, 1), ("morton", 2, 0), ("linear", 8, 0),
                                                ("morton", 8, 1)])
def test_production_trace_per_ray_stores(nbt, ctx, layout, bits, policy):
    """Per-ray parity of the production trace on both layouts, both state widths and both
    outside policies, with perspectives outside the map and corner rays."""
    codes = rand_map(0, 0.3, 0.66, 0.04, seed=21, shape=(33, 41, 47))
    m, om = make_map(nbt, ctx, codes, policy=policy, layout=layout, bits=bits)
    poi = np.array([23.5, 20.5, 16.5])
    P = oracle.sample_perspectives(poi, 35.0, 10, seed=2)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 21, 13)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, 21, 13)
    cam.add_corners = ocam.add_corners = 1
    _per_ray_check(nbt, ctx, m, om, poi, P, cam, ocam, 30.0)


# ---------------------------------------------------------------- frames

def test_frames_bit_exact(nbt, ctx):
    """T19: host (oracle) and device frame quantisation are bit-identical."""
    m, om = make_map(nbt, ctx, np.zeros((4, 4, 4), np.uint8), voxel_size=0.01, origin=(-1.0, 0.5, 0.25))
    rng = np.random.default_rng(0)
    poi = np.array([0.3, 0.9, 0.6])
    P = poi + rng.normal(size=(20000, 3)) * 0.7
    P[:50] = poi + rng.normal(size=(50, 3)) * [1e-9, 1e-9, 1.0]       # near-vertical views (fallback axis)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 640, 480)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, 640, 480)
    q, st = nbt.debug_frames(ctx, m, poi, P, cam, 1.5)
    assert (st == 0).all()
    for i in range(0, len(P), 7):
        f = oracle.frame(om, poi, P[i], ocam, 1.5)
        want = np.concatenate([f[k] for k in ("o", "a", "rh", "uh", "rc", "uc")])
        assert np.array_equal(q[i], want), i


# -------------------------------------------------------------- the ID

def test_config_a_full(nbt, ctx):
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    cloud, g, c = run_both(nbt, ctx, m, om, cfg.poi, P, cfg.width, cfg.height, cfg.range_)
    assert_cloud_equal(cloud, P, g, c)


def test_config_a_every_ray(nbt, ctx):
    """Per-ray parity for config A: device walks of the oracle's endpoints, all 12288 rays."""
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    for p in P:
        o, e, rc = oracle.perspective_rays(om, cfg.poi, p, ocam, cfg.range_)
        _, _, _, cnt = nbt.debug_trace(ctx, m, np.repeat(o[None], len(e), 0), e, 4)
        assert np.array_equal(cnt.astype(np.int64), rc[:, :4])


def test_config_b_subset(nbt, ctx):
    """Config B map, camera and range; every 8th of its 512 perspectives."""
    cfg = CONFIGS["B"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)[::8]
    cloud, g, c = run_both(nbt, ctx, m, om, cfg.poi, P, cfg.width, cfg.height, cfg.range_)
    assert_cloud_equal(cloud, P, g, c)


def test_config_c_two_full_resolution_perspectives(nbt, ctx):
    """640x480 rays (config C) for two perspectives."""
    cfg = CONFIGS["C"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)[[0, 101]]
    cloud, g, c = run_both(nbt, ctx, m, om, cfg.poi, P, cfg.width, cfg.height, cfg.range_)
    assert_cloud_equal(cloud, P, g, c)


def test_config_d_subset(nbt, ctx):
    """512^3 map (config D) at 160x120 rays, 6 of its 4096 perspectives."""
    cfg = CONFIGS["D"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)[::700]
    cloud, g, c = run_both(nbt, ctx, m, om, cfg.poi, P, cfg.width, cfg.height, cfg.range_)
    assert_cloud_equal(cloud, P, g, c)


@pytest.mark.parametrize("w,h,corners", [(1, 1, False), (1, 7, False), (9, 1, True), (13, 5, True), (37, 29, False)])
def test_lattice_shapes(nbt, ctx, w, h, corners):
    """Ragged lattices (not multiples of the 8x4 tile), single rows/columns, corner rays."""
    codes = rand_map(24, 0.3, 0.66, 0.04, seed=w * 7 + h)
    m, om = make_map(nbt, ctx, codes, 0.5, origin=(-1.0, -2.0, 0.5))
    poi = np.array([5.1, 4.2, 6.7])
    P = oracle.sample_perspectives(poi, 4.0, 33, seed=w + h)
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, w, h, 9.0, corners=corners)
    assert_cloud_equal(cloud, P, g, c)


@pytest.mark.parametrize("s_g", [20, 40])
def test_grid_scaling_camera(nbt, ctx, s_g):
    cfg = CONFIGS["B"]
    m, om = make_map(nbt, ctx, syn_map(96, 10.0, 4), 0.01)
    poi = np.array([0.485, 0.485, 0.485])
    P = oracle.sample_perspectives(poi, 0.3, 40, seed=s_g)
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, 0, 0, 0.6, grid=(FOV_H, FOV_V, 0.6, 0.01, float(s_g)))
    assert_cloud_equal(cloud, P, g, c)


@pytest.mark.parametrize("policy", [0, 1])
def test_perspectives_outside_grid(nbt, ctx, policy):
    """Origins outside the map (slow entry path), rays missing the map entirely, clip policy."""
    codes = rand_map(16, 0.3, 0.69, 0.01, seed=11)
    m, om = make_map(nbt, ctx, codes, 1.0, policy=policy)
    poi = np.array([8.0, 8.0, 8.0])
    rng = np.random.default_rng(1)
    d = rng.normal(size=(40, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    P = poi + d * rng.uniform(9, 30, (40, 1))
    P[0] = [-20.0, 8.0, 8.0]
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, 16, 12, 40.0, corners=True)
    assert_cloud_equal(cloud, P, g, c)


def test_degenerate_and_special_maps(nbt, ctx):
    poi = np.array([3.5, 3.5, 3.5])
    m, om = make_map(nbt, ctx, np.full((7, 7, 7), 2, np.uint8), gain=(1.0, 0.12, 0.0))
    P = np.array([[1.0, 1.0, 1.0], [6.0, 2.0, 3.0]])
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, 8, 6, 5.0)
    assert_cloud_equal(cloud, P, g, c)
    assert (cloud.gain == 0).all()
    with pytest.raises(nbt.NbtError) as ei:
        nbt.id_compute(ctx, m, poi, np.array([[1.0, 1.0, 1.0], poi]), nbt.camera_from_fov(1.0, 1.0, 4, 4), 3.0)
    assert ei.value.status == nbt.ERR_DEGENERATE
    with pytest.raises(nbt.NbtError):     # Q16 overflow: rays far beyond +-2^14 voxels
        nbt.id_compute(ctx, m, poi, P, nbt.camera_from_fov(1.0, 1.0, 4, 4), 40000.0)
    ctx.sync()
    tiny, otiny = make_map(nbt, ctx, np.array([[[1]]], np.uint8))
    cloud, g, c = run_both(nbt, ctx, tiny, otiny, np.array([0.5, 0.5, 0.5]), np.array([[0.5, 0.5, 2.5]]), 3, 3, 4.0)
    assert_cloud_equal(cloud, np.array([[0.5, 0.5, 2.5]]), g, c)


def test_voxel_face_origins(nbt, ctx):
    """Perspectives and PoI exactly on voxel faces / corners (exact-tie starts)."""
    codes = rand_map(20, 0.3, 0.7, 0.0, seed=3)
    m, om = make_map(nbt, ctx, codes)
    poi = np.array([10.0, 10.0, 10.0])
    P = np.array([[2.0, 10.0, 10.0], [10.0, 3.0, 10.0], [4.0, 4.0, 4.0], [16.0, 4.0, 10.5], [10.0, 10.0, 2.0]])
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, 9, 9, 12.0, corners=True)
    assert_cloud_equal(cloud, P, g, c)


def test_slices_and_device_io(nbt, ctx):
    """Shards (first, stride) equal rows of the full result; device in/out equals host in/out."""
    import torch
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, 20.0, 50, seed=3)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 24, 18)
    full = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    for first, stride in [(0, 3), (2, 3), (5, 7), (49, 4)]:
        part = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_, first=first, stride=stride)
        assert np.array_equal(part.gain, full.gain[first::stride])
        assert np.array_equal(part.counts, full.counts[first::stride])
    dP = torch.from_numpy(P).cuda()
    out = nbt.empty_cloud(50, device="cuda")
    nbt.id_compute(ctx, m, cfg.poi, dP, cam, cfg.range_, out=out)
    ctx.sync()
    assert np.array_equal(out.gain.cpu().numpy(), full.gain)
    assert np.array_equal(out.counts.cpu().numpy().astype(np.uint64), full.counts)


def _ray_owner(w, h, corners, world):
    """Shard of every ray (row-major k = kk*W + i, then the 4 corner rays), as include/nbt.h
    states for nbt_id_compute_rays: 8x4-pixel tile units (or runs of 32 rays), dealt
    round-robin; corner rays to shard 0."""
    kk, i = np.divmod(np.arange(w * h), w)
    if w >= 8 and h >= 4:
        unit = (kk // 4) * ((w + 7) // 8) + i // 8
    else:
        unit = np.arange(w * h) // 32
    owner = unit % world
    return np.concatenate([owner, np.zeros(4, np.int64)]) if corners else owner


@pytest.mark.parametrize("w,h,corners,worlds", [(24, 17, True, (1, 2, 3, 7)), (5, 3, False, (1, 2, 5)),
                                                (64, 48, False, (2, 8)), (7, 30, True, (3,))])
def test_ray_split_matches_oracle(nbt, ctx, w, h, corners, worlds):
    """Ray shards (SURVEY 8(e) ray split): each shard's integer totals equal the oracle's
    per-ray counts summed over the rays the header assigns it; the shards' sum finalizes to
    the whole ID bit for bit; shards without rays return zeros."""
    import torch
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    n = 9
    P = oracle.sample_perspectives(cfg.poi, 20.0, n, seed=21)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, w, h)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, w, h)
    cam.add_corners = ocam.add_corners = int(corners)
    full = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    per_ray = [oracle.perspective_rays(om, cfg.poi, p, ocam, cfg.range_)[2] for p in P]
    dP = torch.from_numpy(P).cuda()
    for world in worlds:
        owner = _ray_owner(w, h, corners, world)
        total = torch.zeros((n, nbt.ID_TOTALS), dtype=torch.int64, device="cuda")
        for r in range(world):
            t = nbt.id_compute_rays(ctx, m, cfg.poi, P if r % 2 else dP, cam, cfg.range_, r, world)
            ctx.sync()
            want = np.stack([rc[owner == r, :4].sum(0) for rc in per_ray])
            assert np.array_equal(t.cpu().numpy()[:, :4], want), (world, r)
            total += t
        torch.cuda.synchronize()                      # the adds ran on torch's stream
        fin = nbt.id_finalize(ctx, m, cfg.poi, P, cam, cfg.range_, total)
        assert np.array_equal(fin.xyz, P)
        assert np.array_equal(fin.counts, full.counts)
        assert np.array_equal(fin.gain, full.gain)


@pytest.mark.parametrize("layout", ["linear", "morton"])
@pytest.mark.parametrize("range_", [30.0, 16500.0])
def test_ray_split_layouts_and_wide_rays(nbt, ctx, layout, range_):
    """The ray-shard kernel instances of both map layouts and of the 64-bit walk (rays longer
    than the int32 bound of 16383 voxels per axis: perspectives ~8200 voxels outside the map,
    range 16500, narrow FoV): shard totals sum to the whole ID's, which equals the oracle's."""
    import torch
    codes = rand_map(0, 0.35, 0.64, 0.01, seed=11, shape=(40, 44, 48))
    m, om = make_map(nbt, ctx, codes, layout=layout)
    poi = np.array([24.5, 22.5, 20.5])
    wide = range_ > 16000
    P = oracle.sample_perspectives(poi, 8200.0 if wide else 15.0, 6, seed=5, mode=int(wide))
    fh, fv = (0.2, 0.2) if wide else (FOV_H, FOV_V)
    cam = nbt.camera_from_fov(fh, fv, 21, 13)
    ocam = oracle.camera_from_fov(fh, fv, 21, 13)
    _, g, c = oracle.id_compute(om, poi, P, ocam, range_, nthreads=NTHREADS)
    parts = [nbt.id_compute_rays(ctx, m, poi, P, cam, range_, r, 3) for r in range(3)]
    ctx.sync()
    total = sum(parts)
    torch.cuda.synchronize()
    assert np.array_equal(total.cpu().numpy()[:, :4], c)
    fin = nbt.id_finalize(ctx, m, poi, P, cam, range_, total)
    assert np.array_equal(fin.gain, g)


def test_ray_split_fused_into_peer_totals_one_rank(nbt, ctx):
    """nbt_id_compute_rays_gather with one rank: the shard instance's count flushes go through
    the peer-totals path (atomics into the gather buffer) and finalize to the whole ID."""
    import torch
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, 20.0, 7, seed=31)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 24, 17)
    full = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    g = nbt.Gather(ctx, 16, 1, 0)
    for _ in range(2):                                   # the buffer is cleared between calls
        g.zero()
        g.compute_rays(m, cfg.poi, P, cam, cfg.range_)
        ctx.sync()
        t = g.totals(7).clone()
        assert np.array_equal(t.cpu().numpy()[:, :4], full.counts.astype(np.int64))
        fin = nbt.id_finalize(ctx, m, cfg.poi, P, cam, cfg.range_, t)
        assert np.array_equal(fin.gain, full.gain)
    with pytest.raises(nbt.NbtError):                    # 20 x 40 B do not fit 16 x 64 B
        g.compute_rays(m, cfg.poi, oracle.sample_perspectives(cfg.poi, 20.0, 30, seed=1), cam, cfg.range_)
    g.close()


@pytest.mark.parametrize("policy", [0, 1])
def test_ray_split_fused_outside_origins(nbt, ctx, policy):
    """The fused ray split (counts into the peer totals) with perspectives outside the map and
    rays that never enter it: their Unknown visits (outside policy) reach the peer totals, so
    the finalized cloud equals the whole ID and the oracle."""
    codes = rand_map(16, 0.3, 0.69, 0.01, seed=11)
    m, om = make_map(nbt, ctx, codes, 1.0, policy=policy)
    poi = np.array([8.0, 8.0, 8.0])
    rng = np.random.default_rng(1)
    d = rng.normal(size=(9, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    P = poi + d * rng.uniform(9, 30, (9, 1))
    P[0] = [-20.0, 8.0, 8.0]
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 16, 12)
    cam.add_corners = 1
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, 16, 12)
    ocam.add_corners = 1
    _, g_ref, c_ref = oracle.id_compute(om, poi, P, ocam, 40.0, nthreads=NTHREADS)
    g = nbt.Gather(ctx, 16, 1, 0)
    g.zero()
    g.compute_rays(m, poi, P, cam, 40.0)
    ctx.sync()
    t = g.totals(len(P)).clone()
    assert np.array_equal(t.cpu().numpy()[:, :4], c_ref)
    fin = nbt.id_finalize(ctx, m, poi, P, cam, 40.0, t)
    assert np.array_equal(fin.gain, g_ref)
    g.close()


def test_ray_split_prob_map_and_misuse(nbt, ctx):
    """8-bit store: the summed T_G finalizes to the exact Eq. 2 gains; bad shard arguments and
    host totals are rejected."""
    import ctypes
    import torch
    p, obs = _prob_scene((22, 26, 30), seed=5)
    codes, levels = oracle.quantize_prob(p, obs)
    m = nbt.Map(ctx, nbt.map_desc(30, 26, 22, 1.0), prob=True)
    m.upload_prob(p, obs)
    om = oracle.OracleMap(codes, levels=levels)
    poi = np.array([15.5, 13.5, 11.5])
    P = oracle.sample_perspectives(poi, 10.0, 12, seed=4)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 40, 33)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, 40, 33)
    _, g, c, tg = oracle.id_compute(om, poi, P, ocam, 30.0, nthreads=NTHREADS, with_tg=True)
    parts = [nbt.id_compute_rays(ctx, m, poi, P, cam, 30.0, r, 4) for r in range(4)]
    ctx.sync()
    total = sum(parts)
    torch.cuda.synchronize()
    assert np.array_equal(total.cpu().numpy()[:, :4], c)
    assert np.array_equal(total.cpu().numpy()[:, 4], tg)
    fin = nbt.id_finalize(ctx, m, poi, P, cam, 30.0, total)
    assert np.array_equal(fin.gain, g)
    for r, world in [(4, 4), (-1, 2), (0, 0)]:
        with pytest.raises(nbt.NbtError):
            nbt.id_compute_rays(ctx, m, poi, P, cam, 30.0, r, world)
    with pytest.raises(TypeError):
        nbt.id_finalize(ctx, m, poi, P, cam, 30.0, total.cpu())
    host = np.zeros((12, 5), np.uint64)                   # a host array through the raw ABI
    pp = np.ascontiguousarray(poi)
    st = nbt.lib().nbt_id_compute_rays(ctx.h, m.h, ctypes.c_void_p(pp.ctypes.data),
                                       ctypes.c_void_p(P.ctypes.data), 12, 0, 0, 1, ctypes.byref(cam),
                                       30.0, ctypes.c_void_p(host.ctypes.data))
    assert st == 1 and (host == 0).all()


def test_deterministic_and_permutation(nbt, ctx):
    cfg = CONFIGS["A"]
    m, _ = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, 20.0, 64, seed=8)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 32, 24)
    a = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    b = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    perm = np.random.default_rng(0).permutation(64)
    c = nbt.id_compute(ctx, m, cfg.poi, P[perm], cam, cfg.range_)
    assert np.array_equal(a.gain, b.gain) and np.array_equal(a.counts, b.counts)
    assert np.array_equal(a.gain[perm], c.gain)


def test_update_then_compute_snapshot(nbt, ctx):
    """Stream order: an update issued after a compute does not change what it read."""
    import torch
    cfg = CONFIGS["A"]
    codes = cfg.map_codes()
    m, om = make_map(nbt, ctx, codes, cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, 20.0, 16, seed=1)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 32, 24)
    out = nbt.empty_cloud(16, device="cuda")
    nbt.id_compute(ctx, m, cfg.poi, torch.from_numpy(P).cuda(), cam, cfg.range_, out=out)
    ijk = np.argwhere(codes == 1)[:, ::-1].astype(np.int32)[:20000]
    m.update(ijk, np.full(len(ijk), 2, np.uint8))
    ctx.sync()
    _, g, c = oracle.id_compute(om, cfg.poi, P, oracle.camera_from_fov(FOV_H, FOV_V, 32, 24), cfg.range_)
    assert np.array_equal(out.counts.cpu().numpy().astype(np.int64), c)
    after = _apply_in_order(codes, ijk, np.full(len(ijk), 2, np.uint8))
    om2 = oracle.OracleMap(after, voxel_size=cfg.voxel_size)
    cloud2 = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    _, g2, c2 = oracle.id_compute(om2, cfg.poi, P, oracle.camera_from_fov(FOV_H, FOV_V, 32, 24), cfg.range_)
    assert np.array_equal(cloud2.counts.astype(np.int64), c2)


# -------------------------------------------------------------- sampler

@pytest.mark.parametrize("mode", [0, 1])
def test_sampler_matches_oracle(nbt, ctx, mode):
    poi = np.array([0.3, -0.2, 1.1])
    want = oracle.sample_perspectives(poi, 1.0, 20000, seed=77, mode=mode)
    got = nbt.sample_perspectives(ctx, poi, 1.0, 20000, seed=77, mode=mode)
    assert np.abs(got - want).max() < 1e-12
    import torch
    dev = torch.empty((20000, 3), dtype=torch.float64, device="cuda")
    nbt.sample_perspectives(ctx, poi, 1.0, 20000, seed=77, mode=mode, out=dev)
    ctx.sync()
    assert np.array_equal(dev.cpu().numpy(), got)


# -------------------------------------------------------------- IDW

@pytest.mark.parametrize("power_p,normalize", [(2.0, False), (3.0, False), (2.0, True), (1.0, False)])
def test_idw_matches_oracle(nbt, ctx, power_p, normalize):
    rng = np.random.default_rng(int(power_p * 10) + normalize)
    buf = nbt.IdBuffer(ctx, 10, 700)
    entries = []
    for k in range(13):                               # more than N_B: the oldest 3 are evicted
        n = int(rng.integers(1, 700))
        xyz = rng.normal(size=(n, 3)); gain = rng.uniform(0, 4, n)
        buf.push(nbt.IgCloud(xyz, gain, None))
        entries.append((xyz, gain))
    assert len(buf) == 10
    q = rng.normal(size=(1984, 3)) * 1.2
    q[:5] = entries[-1][0][:5]                        # zero distance to the newest entry
    got = buf.query(q, power_p=power_p, normalize=normalize)
    want = oracle.idw_query(entries[-10:], q, power_p=power_p, normalize=normalize)
    assert np.allclose(got, want, rtol=1e-12, atol=0)


def test_idw_zero_distance_exact(nbt, ctx):
    """Q23: a query on a perspective returns that perspective's gain exactly; among
    coincident perspectives the lowest index wins."""
    rng = np.random.default_rng(3)
    xyz = rng.normal(size=(300, 3)); gain = rng.uniform(0, 4, 300)
    xyz[7] = xyz[200]                      # duplicate position: j = 7 must win
    buf = nbt.IdBuffer(ctx, 4, 300)
    buf.push(nbt.IgCloud(xyz, gain, None))
    q = xyz[[0, 7, 200, 299]] + np.array([0.0, 0.0, 1e-12])[None, :] * 0
    got = buf.query(q)
    assert list(got) == [gain[0], gain[7], gain[7], gain[299]]
    assert np.array_equal(got, oracle.idw_query([(xyz, gain)], q))


def test_idw_empty_and_device(nbt, ctx):
    import torch
    buf = nbt.IdBuffer(ctx, 4, 16)
    with pytest.raises(nbt.NbtError) as ei:
        buf.query(np.zeros((1, 3)))
    assert ei.value.status == nbt.ERR_EMPTY
    xyz = torch.randn(16, 3, dtype=torch.float64, device="cuda")
    gain = torch.rand(16, dtype=torch.float64, device="cuda")
    buf.push(nbt.IgCloud(xyz, gain, None))
    q = torch.randn(100, 3, dtype=torch.float64, device="cuda")
    out = torch.empty(100, dtype=torch.float64, device="cuda")
    buf.query(q, out=out)
    ctx.sync()
    want = oracle.idw_query([(xyz.cpu().numpy(), gain.cpu().numpy())], q.cpu().numpy())
    assert np.allclose(out.cpu().numpy(), want, rtol=1e-12)


# --------------------------------------------- full size, bench launch configuration

def test_full_size_config_b_sampled(nbt, ctx):
    """Config B at its full size (512 x 64x48, the bench workload and launch shape): every
    perspective satisfies the closed-form/invariant bounds, and 24 sampled perspectives
    are recomputed one by one by the oracle."""
    import torch
    cfg = CONFIGS["B"]
    codes = cfg.map_codes()
    m, om = make_map(nbt, ctx, codes, cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    out = nbt.empty_cloud(cfg.n_persp, device="cuda")
    nbt.id_compute(ctx, m, cfg.poi, torch.from_numpy(P).cuda(), cam, cfg.range_, out=out)
    ctx.sync()
    counts = out.counts.cpu().numpy()
    gain = out.gain.cpu().numpy()
    ne = cam.num_rays
    assert (counts[:, 2] <= ne).all() and (counts[:, 3] <= counts[:, :3].sum(1)).all()
    assert (gain >= 0).all() and np.isfinite(gain).all()
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    idx = np.linspace(0, cfg.n_persp - 1, 24).astype(int)
    _, g, c = oracle.id_compute(om, cfg.poi, P[idx], ocam, cfg.range_, nthreads=NTHREADS)
    assert np.array_equal(counts[idx].astype(np.int64), c)
    assert np.array_equal(gain[idx], g)


# ------------------------------------------------ 64-bit decision-term variant

def test_walks_very_long_rays_wide_path(nbt, ctx):
    """Segments of 16000+ voxels on one axis run the int64 variant of the same walk."""
    codes = rand_map(40, 0.5, 0.5, 0.0, seed=13)
    m, om = make_map(nbt, ctx, codes)
    rng = np.random.default_rng(5)
    o = np.round(rng.uniform(5, 35, (40, 3)) * Q16).astype(np.int64)
    d = rng.normal(size=(40, 3)) * [0.2, 0.2, 0.2]
    d[:, 0] = -1.0                                       # x dominant, towards -x
    e = np.round(o / Q16 + d * rng.uniform(16100, 16300, (40, 1))) * Q16
    _compare_walks(nbt, ctx, m, om, o.astype(np.int32), e.astype(np.int32), max_visits=64)


@pytest.mark.parametrize("width", [32, 64])
def test_int32_bound_long_rays(nbt, ctx, width):
    """The int32 decision terms at their tight bound (k_id.cu header: exact while every
    |E_a - O_a| < 2^30 - 1 Q16 units, i.e. < 16383 voxels): segments with |D_x| = 2^30 - 2
    (the longest int32 segment) and just below, axis-parallel and diagonal, walked with the
    terms forced to int32 and to int64, equal the oracle; forcing int32 on |D_x| = 2^30 - 1
    is refused.  Also the former 690-720-voxel boundary region, both widths."""
    codes = rand_map(40, 0.45, 0.5, 0.0, seed=23)
    m, om = make_map(nbt, ctx, codes)
    rng = np.random.default_rng(8)
    lim = (1 << 30) - 2
    o, e = [], []
    for k in range(24):
        oo = np.array([int(rng.integers(0, 40 * Q16)) for _ in range(3)], np.int64)
        dx = lim - int(rng.integers(0, 3 * Q16)) if k % 2 else lim
        oo[0] = min(oo[0], lim - dx + 39 * Q16)          # keep E inside (-2^30, 2^30)
        dy = int(rng.integers(-(1 << 29), 1 << 29)) if k % 3 else 0
        dz = int(rng.integers(-(1 << 28), 1 << 28)) if k % 4 else 0
        o.append(oo)
        e.append(oo - np.array([dx, dy, dz], np.int64))
    for L in (690, 699, 700, 701, 719, 720, 721):       # the former int32 switch (round 1)
        oo = np.array([20 * Q16 + 777, 20 * Q16 + 12345, 20 * Q16 + 999], np.int64)
        o.append(oo); e.append(oo + np.array([L * Q16 + 5, -L * Q16 + 3, 0]))
        o.append(oo); e.append(oo + np.array([L * Q16 + 5, L * Q16 // 2 + 11, -L * Q16 // 3 - 7]))
    o, e = np.array(o).astype(np.int32), np.array(e).astype(np.int32)
    assert (np.abs(e.astype(np.int64) - o).max(1) <= lim).all()
    ctx.set_option(nbt.OPT_WALK_WIDTH, width)
    try:
        _compare_walks(nbt, ctx, m, om, o, e, max_visits=96)
        if width == 32:
            too_long = np.array([[39 * Q16, 5 * Q16, 5 * Q16]], np.int32)
            with pytest.raises(nbt.NbtError):
                nbt.debug_trace(ctx, m, too_long, too_long - np.array([[lim + 1, 0, 0]], np.int32), 8)
    finally:
        ctx.set_option(nbt.OPT_WALK_WIDTH, 0)


def test_id_wide_path(nbt, ctx):
    """Rays longer than the int32 bound (range 16500 voxels from perspectives ~8200 voxels
    outside the map, so both ends stay inside the Q16 coordinate range) select the int64
    trace kernel; the ID equals the oracle."""
    codes = rand_map(48, 0.3, 0.69, 0.01, seed=17)
    m, om = make_map(nbt, ctx, codes, 1.0)
    poi = np.array([24.5, 24.5, 24.5])
    P = oracle.sample_perspectives(poi, 8200.0, 5, seed=6, mode=1)
    fov = 0.2                                            # narrow: the far corners stay inside +-2^14 voxels
    cam = nbt.camera_from_fov(fov, fov, 7, 5)            # odd lattice: the centre ray passes the PoI
    ocam = oracle.camera_from_fov(fov, fov, 7, 5)
    cam.add_corners = ocam.add_corners = 1
    cloud = nbt.id_compute(ctx, m, poi, P, cam, 16500.0)
    _, g, c = oracle.id_compute(om, poi, P, ocam, 16500.0, nthreads=NTHREADS)
    assert_cloud_equal(cloud, P, g, c)
    assert c[:, 3].sum() > 0                             # the rays cross the map


# ---------------------------------------------------------------- store layouts

@pytest.mark.parametrize("bits", [2, 8])
@pytest.mark.parametrize("layout", ["linear", "morton"])
def test_layouts_roundtrip_update_and_id(nbt, ctx, layout, bits):
    """Both map store layouts (Morton cube / linear with sentinel shell) and both state
    widths (2-bit codes / one byte per voxel) give identical, oracle-exact results:
    upload/download, last-wins updates, per-ray walks, the ID."""
    # ragged extents whose Morton cube (128^3 with the 16-voxel shell) is < 8x the linear store
    codes = rand_map(0, 0.3, 0.66, 0.04, seed=21, shape=(33, 41, 47))
    m, om = make_map(nbt, ctx, codes, layout=layout, bits=bits)
    assert np.array_equal(m.download(), codes)
    rng = np.random.default_rng(4)
    ijk = np.stack([rng.integers(0, 47, 900), rng.integers(0, 41, 900), rng.integers(0, 33, 900)], 1).astype(np.int32)
    vals = rng.integers(0, 3, 900).astype(np.uint8)
    m.update(ijk, vals)
    codes2 = _apply_in_order(codes, ijk, vals)
    assert np.array_equal(m.download(), codes2)
    om = oracle.OracleMap(codes2)
    o, e = random_segments_q16(1500, -8.0, 54.0, seed=31)
    _compare_walks(nbt, ctx, m, om, o, e)
    poi = np.array([23.5, 20.5, 16.5])
    P = oracle.sample_perspectives(poi, 16.0, 24, seed=2)
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, 20, 14, 30.0, corners=True)
    assert_cloud_equal(cloud, P, g, c)


def test_elongated_map_rejects_morton(nbt, ctx):
    """A map whose Morton cube would be > 8x its linear store: the Morton layout is refused
    (NBT_ERR_INVALID_ARG), the linear layout walks it oracle-exactly."""
    codes = rand_map(0, 0.3, 0.7, 0.0, seed=1, shape=(3, 4, 700))
    with pytest.raises(nbt.NbtError):
        make_map(nbt, ctx, codes, layout="morton")
    m, om = make_map(nbt, ctx, codes)
    assert np.array_equal(m.download(), codes)
    o, e = random_segments_q16(500, -5.0, 20.0, seed=3)
    o[:, 0] *= 30; e[:, 0] *= 30
    _compare_walks(nbt, ctx, m, om, o, e, max_visits=128)


def test_config_e_loop(nbt):
    """Config E receding-horizon loop (tools/config_e.py): 200 cycles of deltas + moving PoI;
    at cycles 0, 100 and 199 the device map replica equals the sensor-side map, and the
    per-state totals and g_P equal the oracle's; the IDW values match the oracle's Eq. 4
    over the same buffered clouds."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import config_e
    history = []
    checked = []

    def on_cycle(t, s):
        history.append((s["persp"].cpu().numpy(), s["cloud"].gain.cpu().numpy()))
        if t not in (0, 100, 199):
            return
        cfg = s["cfg"]
        assert np.array_equal(s["map"].download(), s["codes"])
        om = oracle.OracleMap(s["codes"], voxel_size=cfg.voxel_size)
        ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
        P = s["persp"].cpu().numpy()
        _, g, c = oracle.id_compute(om, s["poi"], P, ocam, cfg.range_, nthreads=NTHREADS)
        assert np.array_equal(s["cloud"].counts.cpu().numpy().astype(np.int64), c)
        assert np.array_equal(s["cloud"].gain.cpu().numpy(), g)
        want = oracle.idw_query(history[-cfg.extra["n_b"]:], s["queries"], power_p=cfg.extra["power_p"])
        assert np.allclose(s["idw"].cpu().numpy(), want, rtol=1e-12)
        checked.append(t)

    dev_ms, _ = config_e.run_loop(200, on_cycle)
    assert checked == [0, 100, 199] and len(dev_ms) == 200


# ------------------------------------------- f2: orientation factor + information cost

@pytest.mark.parametrize("on_device", [False, True])
def test_info_cost_matches_oracle(nbt, ctx, on_device):
    """O(x) bit-exact (same rounded-once expression), G within 1e-12, c_I within 1e-12, for
    64 trajectories of K+1 = 31 poses."""
    import torch
    rng = np.random.default_rng(11)
    poi = np.array([0.3, -0.1, 0.5])
    buf = nbt.IdBuffer(ctx, 10, 512)
    entries = []
    for _ in range(4):
        xyz = poi + rng.normal(size=(512, 3)) * 0.6
        gain = rng.uniform(0, 80, 512)
        buf.push(nbt.IgCloud(xyz, gain, None))
        entries.append((xyz, gain))
    n = 64 * 31
    pos = poi + rng.normal(size=(n, 3)) * 0.8
    axis = (poi - pos) + rng.normal(size=(n, 3)) * 0.4          # mostly towards the PoI
    axis[::7] *= -1.0                                           # some looking away
    cut = math.cos(math.radians(32.5))
    o_ref, g_ref, c_ref = oracle.info_cost(entries, pos, axis, 31, poi, cut, w_i=25.0)
    if on_device:
        tp, ta = torch.from_numpy(pos).cuda(), torch.from_numpy(axis).cuda()
        out = tuple(torch.empty(k, dtype=torch.float64, device="cuda") for k in (n, n, 64))
        buf.info_cost(tp, ta, 31, poi, cut, 25.0, out=out)
        ctx.sync()
        o, g, c = (t.cpu().numpy() for t in out)
    else:
        o, g, c = buf.info_cost(pos, axis, 31, poi, cut, 25.0)
    assert np.array_equal(o, o_ref)
    assert (o == 0).any() and (o > 0).any()
    assert np.allclose(g, g_ref, rtol=1e-12)
    assert np.allclose(c, c_ref, rtol=1e-12)
    with pytest.raises(nbt.NbtError) as ei:
        bad = pos.copy(); bad[5] = poi
        buf.info_cost(bad, axis, 31, poi, cut, 25.0)
    assert ei.value.status == nbt.ERR_DEGENERATE


# ------------------------------------------------------------------ CUDA graphs

def test_graph_capture_replays_the_cycle(nbt):
    """An MHP cycle (deltas -> sampling -> ID -> push -> IDW) captured into CUDA graphs and
    replayed gives exactly the eager results, including the device-side ring buffer."""
    import torch
    cfg = CONFIGS["A"]
    codes = cfg.map_codes()
    rng = np.random.default_rng(0)
    deltas = []
    for _ in range(2):
        ijk = rng.integers(0, cfg.n, (300, 3)).astype(np.int32)
        deltas.append((torch.from_numpy(ijk).cuda(), torch.from_numpy(rng.integers(0, 3, 300).astype(np.uint8)).cuda()))
    q = torch.from_numpy(oracle.sample_perspectives(cfg.poi, 30.0, 200, seed=9)).cuda()
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 24, 18)

    def setup():
        ctx = nbt.Ctx(0)
        m = nbt.Map(ctx, nbt.map_desc(cfg.n, cfg.n, cfg.n, cfg.voxel_size))
        m.upload(codes)
        st = dict(ctx=ctx, m=m, persp=torch.empty((40, 3), dtype=torch.float64, device="cuda"),
                  cloud=nbt.empty_cloud(40, device="cuda"), buf=nbt.IdBuffer(ctx, 3, 40),
                  out=torch.empty(200, dtype=torch.float64, device="cuda"))
        return st

    def cycle(st, c):
        ijk, val = deltas[c % 2]
        st["m"].update(ijk, val)
        nbt.sample_perspectives(st["ctx"], cfg.poi, 20.0, 40, 100 + c % 2, 0, out=st["persp"])
        nbt.id_compute(st["ctx"], st["m"], cfg.poi, st["persp"], cam, cfg.range_, out=st["cloud"])
        st["buf"].push(st["cloud"], 40)
        st["buf"].query(q, out=st["out"])

    def snapshot(st):
        st["ctx"].sync()
        return (st["m"].download(), st["cloud"].counts.cpu().numpy(), st["cloud"].gain.cpu().numpy(),
                st["out"].cpu().numpy())

    A, B = setup(), setup()
    cycle(A, 0); cycle(B, 0)                       # warm-up: sizes every scratch buffer
    graphs = []
    for c in (0, 1):
        B["ctx"].capture_begin()
        cycle(B, c)
        graphs.append(B["ctx"].capture_end())
    for c in range(1, 7):
        cycle(A, c)
        graphs[c % 2].launch()
        for a, b in zip(snapshot(A), snapshot(B)):
            assert np.array_equal(a, b), c
    with pytest.raises(nbt.NbtError) as ei:        # host buffers are refused while capturing
        B["ctx"].capture_begin()
        try:
            nbt.id_compute(B["ctx"], B["m"], cfg.poi, np.zeros((2, 3)), cam, cfg.range_)
        finally:
            B["ctx"].capture_end().close()
    assert ei.value.status == nbt.ERR_STATE


def test_handles_destroyed_in_any_order(nbt):
    """Destroying the ctx before its maps, buffers and graphs defers the release (no crash)."""
    import torch
    ctx = nbt.Ctx(0)
    m = nbt.Map(ctx, nbt.map_desc(8, 8, 8, 1.0))
    buf = nbt.IdBuffer(ctx, 2, 4)
    buf.push(nbt.IgCloud(torch.zeros((4, 3), dtype=torch.float64, device="cuda"),
                         torch.ones(4, dtype=torch.float64, device="cuda"), None), 4)
    ctx.capture_begin()
    buf.push(nbt.IgCloud(torch.zeros((4, 3), dtype=torch.float64, device="cuda"),
                         torch.ones(4, dtype=torch.float64, device="cuda"), None), 4)
    g = ctx.capture_end()
    ctx.close()
    g.launch()
    g.close()
    assert (m.download() == 0).all()
    buf.close()
    m.close()


# ------------------------------------------- f1: per-voxel probability (exact Eq. 2)

def _prob_scene(shape, seed):
    rng = np.random.default_rng(seed)
    codes = rand_map(0, 0.3, 0.65, 0.05, seed=seed, shape=shape)
    p = np.where(codes == 1, rng.uniform(0.12, 0.5, shape), rng.uniform(0.5, 0.97, shape)).astype(np.float32)
    observed = (codes != 0).astype(np.uint8)
    return p, observed


@pytest.mark.parametrize("layout", ["linear", "morton"])
def test_prob_map_id_matches_oracle(nbt, ctx, layout):
    """8-bit store: upload_prob reproduces the oracle's states and levels, and the ID (exact
    Eq. 2 per voxel) matches the oracle bit for bit: per-state totals and g_P."""
    p, obs = _prob_scene((22, 26, 30), seed=5)
    codes, levels = oracle.quantize_prob(p, obs)
    m = nbt.Map(ctx, nbt.map_desc(30, 26, 22, 1.0, layout=layout), prob=True)
    m.upload_prob(p, obs)
    assert np.array_equal(m.download(), codes)
    assert np.array_equal(m.download_levels(), levels)
    om = oracle.OracleMap(codes, levels=levels)
    poi = np.array([15.5, 13.5, 11.5])
    P = oracle.sample_perspectives(poi, 10.0, 30, seed=3)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, 24, 17)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, 24, 17)
    cam.add_corners = ocam.add_corners = 1
    cloud = nbt.id_compute(ctx, m, poi, P, cam, 30.0)
    _, g, c, tg = oracle.id_compute(om, poi, P, ocam, 30.0, nthreads=NTHREADS, with_tg=True)
    assert np.array_equal(cloud.counts.astype(np.int64), c)
    assert np.array_equal(cloud.gain, g)
    assert (tg > 0).all()


def test_prob_map_updates_and_defaults(nbt, ctx):
    """update_prob applies (state, level) deltas in order (last wins); state-only writes store
    P_F = g_F and P_O = 1 - g_O rounded to k/63 (8 and 61 with the default gains)."""
    p, obs = _prob_scene((9, 10, 11), seed=8)
    codes, levels = oracle.quantize_prob(p, obs)
    m = nbt.Map(ctx, nbt.map_desc(11, 10, 9, 1.0), prob=True)
    m.upload_prob(p, obs)
    rng = np.random.default_rng(1)
    n = 700
    ijk = np.stack([rng.integers(0, 11, n), rng.integers(0, 10, n), rng.integers(0, 9, n)], 1).astype(np.int32)
    ijk[n // 2:] = ijk[:n - n // 2]
    dp = rng.uniform(0, 1, n).astype(np.float32)
    dobs = (rng.uniform(size=n) < 0.9).astype(np.uint8)
    m.update_prob(ijk, dp, dobs)
    dc, dl = oracle.quantize_prob(dp, dobs)
    want_c, want_l = codes.copy(), levels.copy()
    for (x, y, z), cc, ll in zip(ijk, dc, dl):
        want_c[z, y, x] = cc
        want_l[z, y, x] = ll
    assert np.array_equal(m.download(), want_c)
    assert np.array_equal(m.download_levels(), want_l)
    m.update(np.array([[1, 2, 3], [4, 5, 6], [7, 8, 0]], np.int32), np.array([1, 2, 0], np.uint8))
    lv = m.download_levels()
    assert (lv[3, 2, 1], lv[6, 5, 4], lv[0, 8, 7]) == (8, 61, 0)
    ctx.sync()


def test_prob_map_walks(nbt, ctx):
    """The 8-bit store walks the same voxels with the same states as the 2-bit store."""
    p, obs = _prob_scene((12, 12, 12), seed=2)
    codes, levels = oracle.quantize_prob(p, obs)
    m = nbt.Map(ctx, nbt.map_desc(12, 12, 12, 1.0), prob=True)
    m.upload_prob(p, obs)
    om = oracle.OracleMap(codes)
    o, e = random_segments_q16(1500, -5.0, 17.0, seed=6)
    _compare_walks(nbt, ctx, m, om, o, e)


def test_byte_store_config_b_subset(nbt, ctx):
    """The byte-per-voxel state store on config B's map and camera: bit-exact vs the oracle."""
    cfg = CONFIGS["B"]
    codes = cfg.map_codes()
    m, om = make_map(nbt, ctx, codes, voxel_size=cfg.voxel_size, bits=8)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, 24, seed=cfg.persp_seed, mode=cfg.persp_mode)
    cloud, g, c = run_both(nbt, ctx, m, om, cfg.poi, P, cfg.width, cfg.height, cfg.range_)
    assert_cloud_equal(cloud, P, g, c)


# ---------------------------------------------------------------- randomized configurations

@pytest.mark.parametrize("seed", range(int(os.environ.get("NBT_FUZZ_SEEDS", "12"))))
def test_random_configurations_fuzz(nbt, ctx, seed):
    """Random non-cubic maps (random voxel size and origin, random codes or SYN), random
    PoI and perspectives (some outside the grid), random lattice shape, corners, range,
    outside policy, gains, layout and state width: the whole ID bit-exact vs the oracle."""
    rng = np.random.default_rng(1000 + seed)
    layout = "morton" if rng.random() < 0.3 else "linear"
    bits = 8 if rng.random() < 0.3 else 2
    nx, ny, nz = (int(v) for v in rng.integers(3, 48, 3))
    s = float(rng.choice([0.01, 0.05, 0.37, 1.0, 2.5]))
    origin = tuple(float(v) for v in rng.uniform(-20, 20, 3) * s)
    if rng.random() < 0.5:
        codes = rand_map(0, *rng.dirichlet([2, 5, 0.5]), seed=seed, shape=(nz, ny, nx))
    else:
        n = int(min(nx, ny, nz))
        codes = syn_map(max(n, 8), max(2.0, n / 6), seed)[:nz, :ny, :nx].copy()
        codes = np.pad(codes, ((0, nz - codes.shape[0]), (0, ny - codes.shape[1]), (0, nx - codes.shape[2])),
                       constant_values=1)
    policy = int(rng.random() < 0.3)
    gain = tuple(float(v) for v in rng.uniform(0, 1, 3))
    try:
        m, om = make_map(nbt, ctx, codes, voxel_size=s, origin=origin, gain=gain, policy=policy, layout=layout,
                         bits=bits)
    except nbt.NbtError:                   # a Morton cube > 8x the store is refused (tested above)
        m, om = make_map(nbt, ctx, codes, voxel_size=s, origin=origin, gain=gain, policy=policy, bits=bits)
    ext = np.array([nx, ny, nz], float) * s
    poi = np.array(origin) + rng.uniform(-0.1, 1.1, 3) * ext
    r_s = float(rng.uniform(0.2, 1.5) * ext.max())
    P = oracle.sample_perspectives(poi, r_s, int(rng.integers(1, 40)), seed=seed, mode=int(rng.integers(0, 2)))
    w, h = int(rng.integers(1, 24)), int(rng.integers(1, 18))
    range_ = float(rng.uniform(0.1, 2.0) * ext.max())
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, w, h, range_, corners=bool(rng.random() < 0.4))
    assert_cloud_equal(cloud, P, g, c)


def test_binding_rejects_mismatched_buffers(nbt, ctx):
    """The binding checks buffer sizes before the C call (no host or device overrun)."""
    import torch
    m, _ = make_map(nbt, ctx, rand_map(0, seed=1, shape=(5, 6, 7)))
    with pytest.raises((nbt.NbtError, ValueError)):
        m.upload(np.zeros(10, np.uint8))
    with pytest.raises(ValueError):
        m.update(np.zeros((3, 3), np.int32), np.zeros(4, np.uint8))
    poi = np.array([3.5, 3.0, 2.5])
    P = np.array([[1.0, 1.0, 1.0], [6.0, 5.0, 4.0]])
    cam = nbt.camera_from_fov(1.0, 1.0, 4, 4)
    with pytest.raises(ValueError):
        nbt.id_compute(ctx, m, poi, P, cam, 5.0, out=nbt.empty_cloud(1))
    with pytest.raises(ValueError):
        nbt.id_compute(ctx, m, poi, P.ravel()[:5], cam, 5.0)
    buf = nbt.IdBuffer(ctx, 2, 4)
    cloud = nbt.id_compute(ctx, m, poi, P, cam, 5.0)
    with pytest.raises(ValueError):
        buf.push(cloud, 3)
    with pytest.raises(ValueError):
        mixed = nbt.IgCloud(torch.from_numpy(cloud.xyz).cuda(), cloud.gain, None)
        buf.push(mixed)
    buf.push(cloud)
    with pytest.raises(ValueError):
        buf.query(np.zeros((4, 3)), out=np.zeros(2))
    with pytest.raises(ValueError):
        nbt.sample_perspectives(ctx, poi, 1.0, 10, 3, out=np.zeros((5, 3)))


def test_large_grid_1024(nbt, ctx):
    """A 1024^3 map (2-bit store 272 MB, beyond L2) with long rays crossing it: walks and the
    ID bit-exact vs the oracle on a handful of perspectives (maximum-size case)."""
    n = 1024
    codes = np.ones((n, n, n), np.uint8)
    codes[:, :, 700:702] = 2                          # an occupied wall
    codes[100:400, 200:600, 300:310] = 0               # an unknown block
    codes[::97, ::89, ::83] = 2                        # sparse occupied voxels
    m, om = make_map(nbt, ctx, codes)
    poi = np.array([512.5, 512.5, 512.5])
    P = np.array([[20.0, 30.0, 40.0], [1000.0, 900.0, 50.0], [512.0, 10.0, 1000.0], [-50.0, 512.0, 512.0]])
    cloud, g, c = run_both(nbt, ctx, m, om, poi, P, 12, 9, 1500.0, corners=True)
    assert_cloud_equal(cloud, P, g, c)
    o, e = random_segments_q16(300, -20.0, 1040.0, seed=77)
    _compare_walks(nbt, ctx, m, om, o, e, max_visits=3200)
    del codes


@pytest.mark.parametrize("knn", [1, 3, 8, 16])
@pytest.mark.parametrize("power_p", [2.0, 3.0])
def test_idw_knn_matches_oracle(nbt, ctx, knn, power_p):
    """Optional k-nearest Eq. 4 (reading Q22) vs the oracle: ragged entries (some smaller
    than knn), an evicting ring, zero-distance queries, equal-distance ties; 1e-12 relative."""
    rng = np.random.default_rng(int(knn * 10 + power_p))
    buf = nbt.IdBuffer(ctx, 6, 600)
    entries = []
    for k in range(8):
        n = int(rng.integers(1, 600)) if k % 3 else int(rng.integers(1, knn + 1))
        xyz = rng.normal(size=(n, 3)); gain = rng.uniform(0, 4, n)
        if n > 4:
            xyz[3] = -xyz[2]                            # equal distance to the origin
        buf.push(nbt.IgCloud(xyz, gain, None))
        entries.append((xyz, gain))
    q = rng.normal(size=(777, 3)) * 1.3
    q[:4] = entries[-1][0][:4]                          # zero distance to the newest entry
    q[4] = 0.0                                          # ties at the origin
    got = buf.query(q, power_p=power_p, knn=knn)
    want = oracle.idw_query_knn(entries[-6:], q, knn, power_p=power_p)
    assert np.allclose(got, want, rtol=1e-12, atol=0)
    # knn = 0 is the full sum
    assert np.allclose(buf.query(q, power_p=power_p, knn=0), oracle.idw_query(entries[-6:], q, power_p=power_p),
                       rtol=1e-12, atol=0)
    with pytest.raises(nbt.NbtError):
        buf.query(q, knn=17)


@pytest.mark.parametrize("name,sampled,bits", [("C'", 3, 2), ("C'", 3, 8), ("D", 5, 2)])
def test_full_size_north_star_and_d_sampled(nbt, ctx, name, sampled, bits):
    """The north-star config C' (512 x 640x480 on 256^3) and config D (4096 x 160x120 on
    512^3) computed whole, in bench.py's launch shape, with sampled perspectives recomputed
    one by one by the oracle: per-state totals and g_P bit-exact."""
    import torch
    cfg = CONFIGS[name]
    codes = cfg.map_codes()
    m, om = make_map(nbt, ctx, codes, cfg.voxel_size, bits=bits)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    out = nbt.empty_cloud(cfg.n_persp, device="cuda")
    nbt.id_compute(ctx, m, cfg.poi, torch.from_numpy(P).cuda(), cam, cfg.range_, out=out)
    ctx.sync()
    counts = out.counts.cpu().numpy()
    gain = out.gain.cpu().numpy()
    assert np.isfinite(gain).all() and (counts[:, 2] <= cam.num_rays).all()
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    idx = np.linspace(0, cfg.n_persp - 1, sampled).astype(int)
    _, g, c = oracle.id_compute(om, cfg.poi, P[idx], ocam, cfg.range_, nthreads=NTHREADS)
    assert np.array_equal(counts[idx].astype(np.int64), c)
    assert np.array_equal(gain[idx], g)


@pytest.mark.parametrize("name,bits,sampled", [("C'", 8, 2), ("D", 2, 5)])
def test_full_size_per_ray_production_trace(nbt, ctx, name, bits, sampled):
    """The production trace kernel at bench.py's full launch (all 512 x 640x480 rays of C' on
    the byte store the bench's C' block uses; all 4096 x 160x120 rays of D on the 2-bit store),
    in its record instance: every ray of sampled perspectives -- (n_U, n_F, n_O, lookups, stop)
    -- equals the oracle's, and every perspective's recorded rays sum to the production
    kernel's totals."""
    import torch
    cfg = CONFIGS[name]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size, bits=bits)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    rays = nbt.debug_id_rays(ctx, m, cfg.poi, P, cam, cfg.range_)
    out = nbt.empty_cloud(cfg.n_persp, device="cuda")
    nbt.id_compute(ctx, m, cfg.poi, torch.from_numpy(P).cuda(), cam, cfg.range_, out=out)
    ctx.sync()
    assert np.array_equal(rays[:, :, :4].sum(1, dtype=np.int64), out.counts.cpu().numpy())
    for j in np.linspace(0, cfg.n_persp - 1, sampled).astype(int):
        _, _, want = oracle.perspective_rays(om, cfg.poi, P[j], ocam, cfg.range_)
        assert np.array_equal(rays[j].astype(np.int64), want), j
    del rays


def test_ctx_options_roundtrip_and_range(nbt, ctx):
    """nbt_ctx_set_option / get_option: defaults, round trip, out-of-range and unknown options
    rejected; a non-default trace tuning gives the same ID bit for bit."""
    assert ctx.get_option(nbt.OPT_TRACE_REFILL_MIN) == 32
    assert ctx.get_option(nbt.OPT_TRACE_CHUNK_MIN) == 64
    assert ctx.get_option(nbt.OPT_WALK_WIDTH) == 0
    for opt, bad in [(nbt.OPT_TRACE_REFILL_MIN, 0), (nbt.OPT_TRACE_REFILL_MIN, 33), (nbt.OPT_TRACE_CHUNK_MIN, 16),
                     (nbt.OPT_TRACE_CARVEOUT, 101), (nbt.OPT_WALK_WIDTH, 48), (nbt.OPT_DELTA_SORT, 2), (99, 0)]:
        with pytest.raises(nbt.NbtError):
            ctx.set_option(opt, bad)
    cfg = CONFIGS["A"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, cfg.n_persp, cfg.persp_seed, cfg.persp_mode)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    ref = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    try:
        ctx.set_option(nbt.OPT_TRACE_REFILL_MIN, 1)
        ctx.set_option(nbt.OPT_TRACE_CHUNK_MIN, 100)
        assert ctx.get_option(nbt.OPT_TRACE_CHUNK_MIN) == 128
        ctx.set_option(nbt.OPT_TRACE_CARVEOUT, 50)
        alt = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
        assert np.array_equal(alt.counts, ref.counts) and np.array_equal(alt.gain, ref.gain)
    finally:
        ctx.set_option(nbt.OPT_TRACE_REFILL_MIN, 32)
        ctx.set_option(nbt.OPT_TRACE_CHUNK_MIN, 64)
        ctx.set_option(nbt.OPT_TRACE_CARVEOUT, 25)


def test_map_extent_limit_of_the_bit_offset_walk(nbt, ctx):
    """The walk addresses the linear 2-bit store by the 32-bit bit offset 2i of a code
    (k_id.cu idx_shift), so that store is refused from a padded extent of 2^31 voxels on
    (NBT_ERR_INVALID_ARG from the descriptor check, before any allocation); the byte store of
    the same extents stays within its own 2^32 limit (checked only, not created: 2.2 GB)."""
    n = 1260                                           # (1260 + 32)^3 = 2.157e9 >= 2^31
    assert (n + 32) ** 3 >= 2 ** 31 and (n + 32) ** 3 < 2 ** 32
    with pytest.raises(nbt.NbtError) as ei:
        nbt.Map(ctx, nbt.map_desc(n, n, n, 0.01))
    assert "2^31" in str(ei.value)
    m = nbt.Map(ctx, nbt.map_desc(1255, 1255, 8, 0.01))   # (1287^2 * 40) < 2^31: accepted
    m.close()


def test_trace_schedules_agree_on_config_b(nbt, ctx):
    """The lockstep walk (default, NBT_OPT_TRACE_REFILL_MIN = 32) and the per-lane refill forms
    (thresholds 1 and 6, the queue instance) give the same integer totals and g_P bit for bit on
    config B's map and camera (64 perspectives), and equal the oracle on a few of them."""
    cfg = CONFIGS["B"]
    m, om = make_map(nbt, ctx, cfg.map_codes(), cfg.voxel_size)
    P = oracle.sample_perspectives(cfg.poi, cfg.persp_radius, 64, cfg.persp_seed, cfg.persp_mode)
    cam = nbt.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    ref = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
    try:
        for thr in (1, 6):
            ctx.set_option(nbt.OPT_TRACE_REFILL_MIN, thr)
            alt = nbt.id_compute(ctx, m, cfg.poi, P, cam, cfg.range_)
            assert np.array_equal(alt.counts, ref.counts) and np.array_equal(alt.gain, ref.gain), thr
    finally:
        ctx.set_option(nbt.OPT_TRACE_REFILL_MIN, 32)
    ocam = oracle.camera_from_fov(FOV_H, FOV_V, cfg.width, cfg.height)
    _, g, c = oracle.id_compute(om, cfg.poi, P[:4], ocam, cfg.range_)
    assert np.array_equal(ref.counts[:4].astype(np.int64), c)
    assert np.array_equal(ref.gain[:4], g)
