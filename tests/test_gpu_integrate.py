"""Map integration on the device vs the CPU oracle, on the same seeded
depth frames: the voxel filter's centroids and counts, the float32 log-odds store, the ID map
states and probability levels, and the emitted a2 deltas must all be bit-exact (every step
is integer, or IEEE operations in the same order on both sides: readings Q33-Q37)."""
import math
import os

import numpy as np
import pytest

import oracle
import nbt_inputs as I

pytestmark = pytest.mark.gpu


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


def same_logodds(a, b):
    """Bit-exact, except that every NaN (never observed) matches every NaN."""
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32))


def oracle_deltas(L0, L1, touched):
    """The (voxel -> (state, level)) changes the oracle's before/after stores imply."""
    c0, l0 = oracle.occ_classify(L0)
    c1, l1 = oracle.occ_classify(L1)
    ch = (touched > 0) & ((c0 != c1) | (l0 != l1))
    zyx = np.argwhere(ch)
    return {(int(x), int(y), int(z)): (int(c1[z, y, x]), int(l1[z, y, x])) for z, y, x in zyx}


def device_deltas(occ):
    ijk, codes, levels = occ.deltas()
    d = {}
    for (x, y, z), c, lv in zip(ijk.tolist(), codes.tolist(), levels.tolist()):
        assert (x, y, z) not in d, "a voxel appears twice in one cloud's deltas"
        d[(x, y, z)] = (c, lv)
    return d


def map_levels_expected(codes, levels):
    """download_levels reports 0 for Unknown voxels."""
    return np.where(codes == 0, 0, levels).astype(np.uint8)


@pytest.mark.parametrize("name", ["F0", "F"])
def test_voxel_filter_matches_oracle(nbt, ctx, name):
    cf = I.CLOUD_CONFIGS[name]
    pts = cf.cloud(1)
    want, wcnt = oracle.voxel_filter(pts, cf.leaf)
    got, gcnt = nbt.voxel_filter(ctx, pts, cf.leaf)
    assert got.shape == want.shape
    assert np.array_equal(gcnt, wcnt)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n", [1, 2, 7, 1000, 65537])
def test_voxel_filter_ragged_and_negative(nbt, ctx, n):
    rng = np.random.default_rng(n)
    pts = rng.normal(0.0, 0.3, (n, 3))
    pts[: n // 3] = np.round(pts[: n // 3] * 40) / 40          # points on cell faces
    want, wcnt = oracle.voxel_filter(pts, 0.025)
    got, gcnt = nbt.voxel_filter(ctx, pts, 0.025)
    assert np.array_equal(gcnt, wcnt) and np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_voxel_filter_device_input_and_errors(nbt, ctx):
    import torch
    pts = I.CLOUD_CONFIGS["F0"].cloud(0)
    want, wcnt = oracle.voxel_filter(pts, 0.04)
    got, gcnt = nbt.voxel_filter(ctx, torch.from_numpy(pts).cuda(), 0.04)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)) and np.array_equal(gcnt, wcnt)
    e, c = nbt.voxel_filter(ctx, np.zeros((0, 3)), 0.1)
    assert e.shape == (0, 3)
    bad = pts.copy()
    bad[5, 1] = np.nan
    with pytest.raises(nbt.NbtError):
        nbt.voxel_filter(ctx, bad, 0.04)
    with pytest.raises(nbt.NbtError):
        nbt.voxel_filter(ctx, np.array([[1e9, 0.0, 0.0]]), 1e-3)   # cell index out of range
    edge = np.array([[32766.5, -32765.5, 0.0], [-32765.25, 32766.75, 5.0]])
    got, gcnt = nbt.voxel_filter(ctx, edge, 1.0)                    # the extreme valid cells
    want, wcnt = oracle.voxel_filter(edge, 1.0)
    assert np.array_equal(got, want) and np.array_equal(gcnt, wcnt)
    with pytest.raises(nbt.NbtError):
        nbt.voxel_filter(ctx, np.array([[0.0, 32767.5, 0.0]]), 1.0)


def _run_sequence(nbt, ctx, cf, n_clouds, prob, layout, params=None, L_start=None, bits=2):
    n = cf.n
    desc = nbt.map_desc(n, n, n, cf.voxel_size, layout=layout, state_bits=bits)
    occ = nbt.OccMap(ctx, desc)
    m = nbt.Map(ctx, desc, prob=prob)
    L = oracle.new_logodds((n, n, n))
    kw = dict(leaf=cf.leaf, max_range=cf.max_range)
    if params:
        kw.update(params)
    if L_start is not None:
        assert not prob
        L[...] = L_start
        occ.upload(L_start)
        c0, _ = oracle.occ_classify(L)
        m.upload(c0)                     # the ID map starts consistent with the store
    prm = nbt.integrate_params(cf.voxel_size, **kw)
    for k in range(n_clouds):
        pts = cf.cloud(k)
        L_before = L.copy()
        touched, nr = oracle.integrate(L, cf.voxel_size, (0, 0, 0), cf.sensor(k), pts, **kw)
        occ.integrate(cf.sensor(k), pts, map=m, params=prm)
        st = occ.stats()
        assert st[0] == len(pts) and st[1] == nr
        assert st[2] == int((touched > 0).sum())
        assert same_logodds(occ.download(), L), f"cloud {k}: log-odds differ"
        want = oracle_deltas(L_before, L, touched)
        got = device_deltas(occ)
        assert st[3] == len(got)
        assert got == want, f"cloud {k}: deltas differ"
    codes, levels = oracle.occ_classify(L)
    assert np.array_equal(m.download(), codes)
    if prob:
        assert np.array_equal(m.download_levels(), map_levels_expected(codes, levels))
    return occ, m, L


@pytest.mark.parametrize("store", ["2bit", "byte", "prob"])
@pytest.mark.parametrize("layout", ["linear", "morton"])
def test_integrate_sequence_small(nbt, ctx, store, layout):
    cf = I.CLOUD_CONFIGS["F0"]
    _run_sequence(nbt, ctx, cf, cf.n_clouds, store == "prob", layout, bits=8 if store == "byte" else 2)


@pytest.mark.parametrize("prob", [False, True])
def test_integrate_sequence_full_size(nbt, ctx, prob):
    """Config F: 256^3 at 1 cm, 640x576 Azure-Kinect-size frames, 3 poses."""
    cf = I.CLOUD_CONFIGS["F"]
    _run_sequence(nbt, ctx, cf, 3, prob, "linear")


def test_integrate_without_filter_and_unlimited_range(nbt, ctx):
    """leaf = 0 (every point is a ray) and max_range <= 0 (the 64-bit DDA variant)."""
    cf = I.CLOUD_CONFIGS["F0"]
    _run_sequence(nbt, ctx, cf, 2, True, "linear", params=dict(leaf=0.0, max_range=0.0))


def test_integrate_from_observed_start_hits_clamps(nbt, ctx):
    """Start from a store with random observed log-odds near the clamps and thresholds."""
    cf = I.CLOUD_CONFIGS["F0"]
    rng = np.random.default_rng(8)
    L0 = rng.choice(np.array([np.nan, 0.0, -0.4054651, 3.4, -1.9, 0.5, -1e-7, 1e-7], np.float32),
                    size=(cf.n,) * 3).astype(np.float32)
    _run_sequence(nbt, ctx, cf, 2, False, "linear", L_start=L0)


def test_integrate_sensor_and_points_outside_grid(nbt, ctx):
    """A sensor outside the grid, points on both sides: only in-grid voxels change."""
    cf = I.CloudConfig("Fo", 40, 0.05, 3.0, 96, 80, 1.6, 2, 0.05, 3.0, 5)
    _run_sequence(nbt, ctx, cf, 2, True, "linear")


def test_integrate_zero_points_and_bad_cloud(nbt, ctx):
    cf = I.CLOUD_CONFIGS["F0"]
    desc = nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size)
    occ = nbt.OccMap(ctx, desc)
    m = nbt.Map(ctx, desc)
    occ.integrate(cf.sensor(0), np.zeros((0, 3)), map=m)
    assert occ.stats() == (0, 0, 0, 0)
    assert np.isnan(occ.download()).all()
    pts = cf.cloud(0)
    occ.integrate(cf.sensor(0), pts, map=m, params=nbt.integrate_params(cf.voxel_size, leaf=cf.leaf))
    before = occ.download()
    codes_before = m.download()
    bad = pts.copy()
    bad[100] = [np.inf, 0.0, 0.0]
    occ.integrate(cf.sensor(1), bad, map=m)
    with pytest.raises(nbt.NbtError):
        occ.stats()
    assert same_logodds(occ.download(), before) and np.array_equal(m.download(), codes_before)
    # the flags were cleared: the next good cloud matches the oracle
    L = before.copy()
    oracle.integrate(L, cf.voxel_size, (0, 0, 0), cf.sensor(1), pts, leaf=cf.voxel_size, max_range=5.0)
    occ.integrate(cf.sensor(1), pts, map=m)
    occ.stats()
    assert same_logodds(occ.download(), L)


def test_integrate_device_points_and_id_after(nbt, ctx):
    """Device-resident frames; the integrated map then feeds the ID (the f3 -> a7 chain),
    whose result equals the oracle's ID on the oracle-integrated map."""
    import torch
    cf = I.CLOUD_CONFIGS["F0"]
    desc = nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size)
    occ = nbt.OccMap(ctx, desc)
    m = nbt.Map(ctx, desc)
    L = oracle.new_logodds((cf.n,) * 3)
    for k in range(cf.n_clouds):
        pts = cf.cloud(k)
        oracle.integrate(L, cf.voxel_size, (0, 0, 0), cf.sensor(k), pts, leaf=cf.leaf, max_range=cf.max_range)
        occ.integrate(cf.sensor(k), torch.from_numpy(pts).cuda(), map=m,
                      params=nbt.integrate_params(cf.voxel_size, leaf=cf.leaf, max_range=cf.max_range))
    ctx.sync()
    codes, _ = oracle.occ_classify(L)
    assert np.array_equal(m.download(), codes)
    om = oracle.OracleMap(codes, voxel_size=cf.voxel_size)
    poi = cf.poi
    persp = oracle.sample_perspectives(poi, 0.5, 24, 3, 1)
    cam = nbt.camera_from_fov(I.FOV_H, I.FOV_V, 16, 12)
    cloud = nbt.id_compute(ctx, m, poi, persp, cam, 1.0)
    ocam = oracle.camera_from_fov(I.FOV_H, I.FOV_V, 16, 12)
    xyz, g, c = oracle.id_compute(om, poi, persp, ocam, 1.0)
    assert np.array_equal(cloud.counts.astype(np.int64), c)
    assert np.array_equal(cloud.gain, g)


def test_integrate_exact_ties_and_long_rays(nbt, ctx):
    """Rays whose ends sit on voxel faces, edges and corners (exact ties in the DDA) and long
    rays cut into many pieces: sensor on a voxel corner, points on the Q16 lattice, no
    filter, unlimited range (64-bit walk) and a 3-voxel range (int32 walk)."""
    n = 48
    rng = np.random.default_rng(12)
    sensor = np.array([20.0, 17.0, 23.0])
    pts = np.concatenate([
        rng.integers(-30, n + 30, (3000, 3)).astype(np.float64),                    # corners
        rng.integers(-30, n + 30, (3000, 3)) + rng.integers(0, 2, (3000, 3)) * 0.5,  # faces / edges
        sensor + rng.normal(0, 1, (500, 3)) * np.array([1.0, 0.0, 0.0]),          # axis-parallel
        rng.uniform(-40, n + 40, (3000, 3))])
    for mr in (0.0, 3.0, 30.0):
        L = oracle.new_logodds((n, n, n))
        touched, _ = oracle.integrate(L, 1.0, (0, 0, 0), sensor, pts, leaf=0.0, max_range=mr)
        desc = nbt.map_desc(n, n, n, 1.0)
        occ = nbt.OccMap(ctx, desc)
        occ.integrate(sensor, pts, params=nbt.integrate_params(1.0, leaf=0.0, max_range=mr))
        assert occ.stats()[2] == int((touched > 0).sum())
        assert same_logodds(occ.download(), L), f"max_range {mr}"


def test_integrate_few_dense_cells(nbt, ctx):
    """Degenerate grouping: 400 k points in a handful of filter cells (a coarse leaf, and a
    cloud of identical points) -- bit-exact centroids and store, and fast (the grouping must
    not be quadratic in the points per cell)."""
    import time
    n = 40
    rng = np.random.default_rng(3)
    sensor = np.array([2.0, 3.0, 4.0])
    blob = np.array([30.0, 25.0, 20.0]) + rng.normal(0, 3.0, (400_000, 3))
    same = np.tile(np.array([[31.3, 11.7, 8.2]]), (400_000, 1))
    for pts, leaf in ((blob, 16.0), (same, 1.0)):
        want, wcnt = oracle.voxel_filter(pts, leaf)
        got, gcnt = nbt.voxel_filter(ctx, pts, leaf)
        assert np.array_equal(gcnt, wcnt) and np.array_equal(got.view(np.uint64), want.view(np.uint64))
        L = oracle.new_logodds((n, n, n))
        oracle.integrate(L, 1.0, (0, 0, 0), sensor, pts, leaf=leaf, max_range=0.0)
        occ = nbt.OccMap(ctx, nbt.map_desc(n, n, n, 1.0))
        prm = nbt.integrate_params(1.0, leaf=leaf, max_range=0.0)
        occ.integrate(sensor, pts, params=prm)                     # warm-up
        occ = nbt.OccMap(ctx, nbt.map_desc(n, n, n, 1.0))
        t0 = time.perf_counter()
        occ.integrate(sensor, pts, params=prm)
        ctx.sync()
        dt = time.perf_counter() - t0
        assert same_logodds(occ.download(), L)
        # a quadratic grouping of 400 k points per cell would take minutes; the bound leaves room
        # for the host-side copies on a busy box (0.34 s seen once against ~0.1 s typical)
        assert dt < 1.0, f"{dt:.3f} s for one frame"


@pytest.mark.parametrize("seed", range(int(os.environ.get("NBT_FUZZ_SEEDS", "8"))))
def test_integrate_random_configurations_fuzz(nbt, ctx, seed):
    """Random non-cubic grids (voxel size, origin), sensors inside or outside, random point
    clouds (Gaussian blobs, uniform, on the Q16 lattice), random leaf / range / probabilities /
    thresholds, random start store, layout and store kind: log-odds, deltas and the ID map
    bit-exact vs the oracle over 3 clouds."""
    rng = np.random.default_rng(2000 + seed)
    layout = "morton" if rng.random() < 0.3 else "linear"
    store = rng.choice(["2bit", "byte", "prob"])
    nx, ny, nz = (int(v) for v in rng.integers(4, 40, 3))
    s = float(rng.choice([0.02, 0.1, 0.5, 1.0]))
    origin = tuple(float(v) for v in rng.uniform(-10, 10, 3) * s)
    ext = np.array([nx, ny, nz], float) * s
    desc = nbt.map_desc(nx, ny, nz, s, origin, layout=layout, state_bits=8 if store == "byte" else 2)
    occ = nbt.OccMap(ctx, desc)
    try:
        m = nbt.Map(ctx, desc, prob=store == "prob")
    except nbt.NbtError:               # a Morton cube > 8x the store is refused (test_elongated_map_rejects_morton)
        desc.layout = nbt.LAYOUT_LINEAR
        m = nbt.Map(ctx, desc, prob=store == "prob")
    kw = dict(leaf=float(rng.choice([0.0, s, 0.5 * s, 2.7 * s])),
              max_range=float(rng.choice([0.0, 0.3, 1.0]) * ext.max()),
              p_hit=float(rng.uniform(0.55, 0.95)), p_miss=float(rng.uniform(0.05, 0.45)),
              p_min=float(rng.uniform(0.05, 0.3)), p_max=float(rng.uniform(0.7, 0.99)))
    t_occ = float(rng.uniform(0.4, 0.7))
    t_free = float(min(t_occ, rng.uniform(0.3, 0.5)))
    L = oracle.new_logodds((nz, ny, nx))
    prm = nbt.integrate_params(s, **kw, t_occ=t_occ, t_free=t_free)
    for k in range(3):
        sensor = np.array(origin) + rng.uniform(-0.2, 1.2, 3) * ext
        n = int(rng.integers(0, 4000))
        kind = rng.integers(0, 3)
        if kind == 0:
            pts = sensor + rng.normal(0, 0.4, (n, 3)) * ext
        elif kind == 1:
            pts = np.array(origin) + rng.uniform(-0.3, 1.3, (n, 3)) * ext
        else:
            pts = np.array(origin) + np.round(rng.uniform(-0.3, 1.3, (n, 3)) * ext / s * 2) * s / 2
        L_before = L.copy()
        touched, nr = oracle.integrate(L, s, origin, sensor, pts, **kw)
        occ.integrate(sensor, pts, map=m, params=prm)
        st = occ.stats()
        assert st[1] == nr and st[2] == int((touched > 0).sum())
        assert same_logodds(occ.download(), L), f"cloud {k}"
        c0, l0 = oracle.occ_classify(L_before, t_occ, t_free)
        c1, l1 = oracle.occ_classify(L, t_occ, t_free)
        ch = (touched > 0) & ((c0 != c1) | (l0 != l1))
        want = {(int(x), int(y), int(z)): (int(c1[z, y, x]), int(l1[z, y, x])) for z, y, x in np.argwhere(ch)}
        assert device_deltas(occ) == want
    codes, levels = oracle.occ_classify(L, t_occ, t_free)
    assert np.array_equal(m.download(), codes)
    if store == "prob":
        assert np.array_equal(m.download_levels(), map_levels_expected(codes, levels))


def test_integrate_sorted_filter_path_matches(nbt, ctx):
    """The sort-based voxel filter (option NBT_OPT_FILTER_SORT, the experiment knob) integrates
    to the same store as the default hashed grouping (both bit-exact vs the oracle)."""
    ctx.set_option(nbt.OPT_FILTER_SORT, 1)
    try:
        cf = I.CLOUD_CONFIGS["F0"]
        _run_sequence(nbt, ctx, cf, 2, True, "linear")
    finally:
        ctx.set_option(nbt.OPT_FILTER_SORT, 0)


def test_integrate_captured_in_a_graph(nbt, ctx):
    """Map integration of device-resident frames captured once into a CUDA graph and replayed
    with new frame contents (same size, same sensor pose): bit-exact vs the oracle."""
    import torch
    cf = I.CLOUD_CONFIGS["F0"]
    desc = nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size)
    gctx = nbt.Ctx(0)
    occ = nbt.OccMap(gctx, desc)
    m = nbt.Map(gctx, desc)
    prm = nbt.integrate_params(cf.voxel_size, leaf=cf.leaf, max_range=cf.max_range)
    sensor = cf.sensor(0)
    clouds = [cf.cloud(k) for k in range(3)]
    n = min(len(c) for c in clouds)
    dev_pts = torch.from_numpy(np.ascontiguousarray(clouds[0][:n])).cuda()
    L = oracle.new_logodds((cf.n,) * 3)
    oracle.integrate(L, cf.voxel_size, (0, 0, 0), sensor, clouds[0][:n], leaf=cf.leaf, max_range=cf.max_range)
    occ.integrate(sensor, dev_pts, map=m, params=prm)          # warm-up: scratch buffers grow
    gctx.sync()
    gctx.capture_begin()
    occ.integrate(sensor, dev_pts, map=m, params=prm)
    g = gctx.capture_end()
    for k in (1, 2):
        dev_pts.copy_(torch.from_numpy(np.ascontiguousarray(clouds[k][:n])))
        torch.cuda.synchronize()
        g.launch()
        gctx.sync()
        oracle.integrate(L, cf.voxel_size, (0, 0, 0), sensor, clouds[k][:n], leaf=cf.leaf, max_range=cf.max_range)
        assert same_logodds(occ.download(), L), f"replay {k}"
    codes, _ = oracle.occ_classify(L)
    assert np.array_equal(m.download(), codes)
    g.close(); occ.close(); m.close(); gctx.close()


def test_integrate_api_misuse(nbt, ctx):
    """Errors are reported, not crashed on: a map of another grid, wrong sizes, bad
    parameters, host input during capture, counters during capture."""
    cf = I.CLOUD_CONFIGS["F0"]
    occ = nbt.OccMap(ctx, nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size))
    other = nbt.Map(ctx, nbt.map_desc(cf.n + 1, cf.n, cf.n, cf.voxel_size))
    pts = cf.cloud(0)[:1000]
    with pytest.raises(nbt.NbtError) as ei:
        occ.integrate(cf.sensor(0), pts, map=other)
    assert ei.value.status == nbt.ERR_STATE
    with pytest.raises(nbt.NbtError):
        occ.upload(np.zeros(10, np.float32))
    with pytest.raises(nbt.NbtError):
        occ.integrate(cf.sensor(0), pts, params=nbt.integrate_params(cf.voxel_size, p_hit=1.0))
    with pytest.raises(nbt.NbtError):
        occ.integrate(cf.sensor(0), pts, params=nbt.integrate_params(cf.voxel_size, leaf=-1.0))
    with pytest.raises(nbt.NbtError):
        occ.integrate((np.nan, 0.0, 0.0), pts)
    with pytest.raises(nbt.NbtError):
        nbt.voxel_filter(ctx, pts, 0.0)
    gctx = nbt.Ctx(0)
    occ2 = nbt.OccMap(gctx, nbt.map_desc(cf.n, cf.n, cf.n, cf.voxel_size))
    gctx.capture_begin()
    with pytest.raises(nbt.NbtError) as ei:
        occ2.integrate(cf.sensor(0), pts)                       # host points while capturing
    assert ei.value.status == nbt.ERR_STATE
    with pytest.raises(nbt.NbtError):
        occ2.stats()
    gctx.capture_end().close()
    occ.integrate(cf.sensor(0), pts)                            # the original store still works
    assert occ.stats()[0] == 1000
    occ2.close(); gctx.close()
