"""CPU oracle for the online local Information Distribution -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2503_22588_b200``, ``libnbt.so``) never imports, links or executes it;
the two share no code.  The arithmetic lives in ``oracle/oracle.c`` (plain C,
fp64, -ffp-contract=off), each function citing the PAPER.md passage it follows;
this module is ctypes marshalling only.  ``oracle/exact.py`` is an independent
exact-rational brute-force checker used to pin the DDA.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_INVALID_ARG, ERR_DEGENERATE, ERR_EMPTY, ERR_SELFCHECK = 0, 1, 2, 3, 9


class OracleError(RuntimeError):
    def __init__(self, code, what=""):
        super().__init__(f"oracle error {code} {what}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Map(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("voxel_size", C.c_double), ("origin", C.c_double * 3), ("gain", C.c_double * 3),
                ("outside_policy", C.c_int32), ("codes", C.POINTER(C.c_uint8)), ("levels", C.POINTER(C.c_uint8))]


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("add_corners", C.c_int32),
                ("tan_half_fov_h", C.c_double), ("tan_half_fov_v", C.c_double)]


class Ray(C.Structure):
    _fields_ = [("n_u", C.c_int64), ("n_f", C.c_int64), ("n_o", C.c_int64), ("lookups", C.c_int64),
                ("visits", C.c_int64), ("g63", C.c_int64), ("g", C.c_double), ("stop", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        dp, ip, i64p, u8p = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint8)
        L.orc_camera_from_fov.argtypes = [C.c_double, C.c_double, C.c_int32, C.c_int32, C.POINTER(Camera)]
        L.orc_camera_from_grid_scaling.argtypes = [C.c_double] * 5 + [C.POINTER(Camera)]
        L.orc_camera_num_rays.argtypes = [C.POINTER(Camera)]
        L.orc_camera_num_rays.restype = C.c_int32
        L.orc_trace_ray.argtypes = [C.POINTER(Map), ip, ip, C.c_int32, ip, u8p, ip, C.POINTER(Ray)]
        L.orc_id_compute.argtypes = [C.POINTER(Map), dp, dp, C.c_int32, C.POINTER(Camera), C.c_double,
                                     C.c_int32, dp, dp, i64p, i64p, ip]
        L.orc_perspective_rays.argtypes = [C.POINTER(Map), dp, dp, C.POINTER(Camera), C.c_double, ip, ip, i64p]
        L.orc_frame_export.argtypes = [C.POINTER(Map), dp, dp, C.POINTER(Camera), C.c_double, ip, dp]
        L.orc_idw_query.argtypes = [C.c_int32, ip, C.POINTER(dp), C.POINTER(dp), dp, C.c_int32, C.c_double,
                                    C.c_double, C.c_int32, dp]
        L.orc_idw_query_knn.argtypes = [C.c_int32, ip, C.POINTER(dp), C.POINTER(dp), dp, C.c_int32, C.c_double,
                                        C.c_double, C.c_int32, C.c_int32, dp]
        L.orc_philox4x32.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_philox4x32.restype = None
        L.orc_sample_perspectives.argtypes = [dp, C.c_double, C.c_int32, C.c_uint64, C.c_int32, dp]
        L.orc_eq1.argtypes = [dp, C.c_double, dp, C.c_double, dp]
        L.orc_eq1.restype = None
        L.orc_classify.argtypes = [C.POINTER(C.c_float), u8p, C.c_int64, C.c_double, C.c_double, u8p]
        L.orc_classify.restype = None
        L.orc_quantize_prob.argtypes = [C.POINTER(C.c_float), u8p, C.c_int64, C.c_double, C.c_double, u8p, u8p]
        L.orc_quantize_prob.restype = None
        L.orc_map_update.argtypes = [u8p, C.c_int32, C.c_int32, C.c_int32, ip, u8p, C.c_int64]
        L.orc_orientation_factor.argtypes = [dp, dp, dp, C.c_double, dp]
        L.orc_info_cost.argtypes = [C.c_int32, ip, C.POINTER(dp), C.POINTER(dp), dp, dp, C.c_int32, C.c_int32, dp,
                                    C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32, dp, dp, dp]
        fp = C.POINTER(C.c_float)
        L.orc_voxel_filter.argtypes = [dp, C.c_int64, C.c_double, dp, ip, i64p]
        L.orc_integrate.argtypes = [fp, C.c_int32, C.c_int32, C.c_int32, C.c_double, dp, dp, dp, C.c_int64,
                                    C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                    u8p, i64p]
        L.orc_occ_classify.argtypes = [fp, C.c_int64, C.c_double, C.c_double, u8p, u8p]
        L.orc_occ_classify.restype = None
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _d(a):
    return _p(a, C.c_double)


class OracleMap:
    """Keeps the code array alive while the C struct points into it."""

    def __init__(self, codes_zyx, voxel_size=1.0, origin=(0.0, 0.0, 0.0), gain=(1.0, 0.12, 0.03),
                 outside_policy=0, levels=None):
        """levels (uint8, 0..63, same shape) switches on the per-voxel probability P = level/63."""
        self.codes = np.ascontiguousarray(codes_zyx, dtype=np.uint8)
        self.levels = None if levels is None else np.ascontiguousarray(levels, dtype=np.uint8)
        nz, ny, nx = self.codes.shape
        self.s = Map(nx, ny, nz, float(voxel_size), (C.c_double * 3)(*origin), (C.c_double * 3)(*gain),
                     int(outside_policy), _p(self.codes, C.c_uint8),
                     _p(self.levels, C.c_uint8) if self.levels is not None else None)


def camera_from_fov(fov_h, fov_v, w, h) -> Camera:
    cam = Camera()
    st = lib().orc_camera_from_fov(fov_h, fov_v, w, h, C.byref(cam))
    if st:
        raise OracleError(st, "camera_from_fov")
    return cam


def camera_from_grid_scaling(fov_h, fov_v, range_, voxel_size, s_g) -> Camera:
    cam = Camera()
    st = lib().orc_camera_from_grid_scaling(fov_h, fov_v, range_, voxel_size, s_g, C.byref(cam))
    if st:
        raise OracleError(st, "camera_from_grid_scaling")
    return cam


def num_rays(cam: Camera) -> int:
    return lib().orc_camera_num_rays(C.byref(cam))


def trace_ray(m: OracleMap, o_q16, e_q16, max_visits=4096):
    """One ray: returns (visited ijk [k,3], codes [k] (255 = outside), Ray counts)."""
    o = np.ascontiguousarray(o_q16, dtype=np.int32)
    e = np.ascontiguousarray(e_q16, dtype=np.int32)
    ijk = np.zeros((max_visits, 3), np.int32)
    codes = np.zeros(max_visits, np.uint8)
    n = C.c_int32()
    r = Ray()
    st = lib().orc_trace_ray(C.byref(m.s), _p(o, C.c_int32), _p(e, C.c_int32), max_visits,
                             _p(ijk, C.c_int32), _p(codes, C.c_uint8), C.byref(n), C.byref(r))
    if st:
        raise OracleError(st, "trace_ray")
    k = min(n.value, max_visits)
    return ijk[:k].copy(), codes[:k].copy(), r


def id_compute(m: OracleMap, poi, persp_xyz, cam: Camera, range_, nthreads=1, with_tg=False):
    """The whole ID: returns (xyz [n,3], gain [n], counts [n,4] = T_U,T_F,T_O,lookups)
    (+ tg [n] = 63 * sum of g_R in the per-voxel-probability mode if with_tg)."""
    poi = np.ascontiguousarray(poi, dtype=np.float64)
    P = np.ascontiguousarray(persp_xyz, dtype=np.float64).reshape(-1, 3)
    n = P.shape[0]
    xyz = np.zeros((n, 3)); gain = np.zeros(n); counts = np.zeros((n, 4), np.int64); tg = np.zeros(n, np.int64)
    bad = C.c_int32(-1)
    st = lib().orc_id_compute(C.byref(m.s), _d(poi), _d(P), n, C.byref(cam), float(range_), int(nthreads),
                              _d(xyz), _d(gain), _p(counts, C.c_int64), _p(tg, C.c_int64), C.byref(bad))
    if st:
        raise OracleError(st, f"id_compute (perspective {bad.value})")
    return (xyz, gain, counts, tg) if with_tg else (xyz, gain, counts)


def perspective_rays(m: OracleMap, poi, p, cam: Camera, range_, with_counts=True):
    """Per-ray data of one perspective: (O q16 [3], E q16 [ne,3], counts [ne,5] U,F,O,lookups,stop)."""
    poi = np.ascontiguousarray(poi, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    ne = num_rays(cam)
    o = np.zeros(3, np.int32); e = np.zeros((ne, 3), np.int32)
    rc = np.zeros((ne, 5), np.int64)
    st = lib().orc_perspective_rays(C.byref(m.s), _d(poi), _d(p), C.byref(cam), float(range_),
                                    _p(o, C.c_int32), _p(e, C.c_int32),
                                    _p(rc, C.c_int64) if with_counts else None)
    if st:
        raise OracleError(st, "perspective_rays")
    return o, e, rc


def frame(m: OracleMap, poi, p, cam: Camera, range_):
    """Q16 frame (dict of o,a,rh,uh,rc,uc int32[3]) and fwd/right/up unit vectors."""
    poi = np.ascontiguousarray(poi, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    q = np.zeros(18, np.int32); ax = np.zeros(9)
    st = lib().orc_frame_export(C.byref(m.s), _d(poi), _d(p), C.byref(cam), float(range_),
                                _p(q, C.c_int32), _d(ax))
    if st:
        raise OracleError(st, "frame")
    names = ["o", "a", "rh", "uh", "rc", "uc"]
    out = {k: q[3 * i:3 * i + 3].copy() for i, k in enumerate(names)}
    out.update(fwd=ax[0:3].copy(), right=ax[3:6].copy(), up=ax[6:9].copy())
    return out


def idw_query(entries, queries, power_p=2.0, zero_eps=1e-9, normalize=False):
    """Eq. 4 over entries [(xyz [n,3], gain [n]), ...] oldest -> newest."""
    ents = [(np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3), np.ascontiguousarray(g, dtype=np.float64))
            for x, g in entries]
    sizes = np.array([len(g) for _, g in ents], np.int32)
    xs = (C.POINTER(C.c_double) * max(1, len(ents)))(*[_d(x) for x, _ in ents])
    gs = (C.POINTER(C.c_double) * max(1, len(ents)))(*[_d(g) for _, g in ents])
    q = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(q.shape[0])
    st = lib().orc_idw_query(len(ents), _p(sizes, C.c_int32), xs, gs, _d(q), q.shape[0], float(power_p),
                             float(zero_eps), int(bool(normalize)), _d(out))
    if st:
        raise OracleError(st, "idw_query")
    return out


def idw_query_knn(entries, queries, knn, power_p=2.0, zero_eps=1e-9, normalize=False):
    """Eq. 4 over the knn nearest perspectives of each entry (reading Q22)."""
    ents = [(np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3), np.ascontiguousarray(g, dtype=np.float64))
            for x, g in entries]
    sizes = np.array([len(g) for _, g in ents], np.int32)
    xs = (C.POINTER(C.c_double) * max(1, len(ents)))(*[_d(x) for x, _ in ents])
    gs = (C.POINTER(C.c_double) * max(1, len(ents)))(*[_d(g) for _, g in ents])
    q = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(q.shape[0])
    st = lib().orc_idw_query_knn(len(ents), _p(sizes, C.c_int32), xs, gs, _d(q), q.shape[0], float(power_p),
                                 float(zero_eps), int(bool(normalize)), int(knn), _d(out))
    if st:
        raise OracleError(st, "idw_query_knn")
    return out


def philox4x32(ctr, key):
    c = (C.c_uint32 * 4)(*ctr); k = (C.c_uint32 * 2)(*key); o = (C.c_uint32 * 4)()
    lib().orc_philox4x32(c, k, o)
    return list(o)


def sample_perspectives(poi, r_s, n, seed, mode=0):
    poi = np.ascontiguousarray(poi, dtype=np.float64)
    out = np.zeros((n, 3))
    st = lib().orc_sample_perspectives(_d(poi), float(r_s), int(n), int(seed), int(mode), _d(out))
    if st:
        raise OracleError(st, "sample_perspectives")
    return out


def eq1(poi, r_s, X, x_r):
    poi = np.ascontiguousarray(poi, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.zeros(3)
    lib().orc_eq1(_d(poi), float(r_s), _d(X), float(x_r), _d(out))
    return out


def classify(p, observed, t_occ=0.5, t_free=0.5):
    p = np.ascontiguousarray(p, dtype=np.float32).ravel()
    obs = np.ascontiguousarray(observed, dtype=np.uint8).ravel()
    out = np.zeros(p.size, np.uint8)
    lib().orc_classify(_p(p, C.c_float), _p(obs, C.c_uint8), p.size, float(t_occ), float(t_free),
                       _p(out, C.c_uint8))
    return out


def map_update(m: OracleMap, ijk, vals):
    """Apply deltas in order to the oracle map's code array (in place)."""
    ijk = np.ascontiguousarray(ijk, dtype=np.int32).reshape(-1, 3)
    vals = np.ascontiguousarray(vals, dtype=np.uint8)
    nz, ny, nx = m.codes.shape
    st = lib().orc_map_update(_p(m.codes, C.c_uint8), nx, ny, nz, _p(ijk, C.c_int32), _p(vals, C.c_uint8), len(vals))
    if st:
        raise OracleError(st, "map_update")


def orientation_factor(pos, axis, poi, cos_cut):
    pos, axis, poi = (np.ascontiguousarray(v, dtype=np.float64) for v in (pos, axis, poi))
    o = C.c_double()
    st = lib().orc_orientation_factor(_d(pos), _d(axis), _d(poi), float(cos_cut), C.byref(o))
    if st:
        raise OracleError(st, "orientation_factor")
    return o.value


def info_cost(entries, pos, axis, per, poi, cos_cut, w_i, eps=1e-7, power_p=2.0, zero_eps=1e-9, normalize=False):
    """(O [n], G [n], c_I [n_traj]) for n = n_traj * per poses (trajectories of `per` poses)."""
    ents = [(np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3), np.ascontiguousarray(g, dtype=np.float64))
            for x, g in entries]
    sizes = np.array([len(g) for _, g in ents], np.int32)
    xs = (C.POINTER(C.c_double) * max(1, len(ents)))(*[_d(x) for x, _ in ents])
    gs = (C.POINTER(C.c_double) * max(1, len(ents)))(*[_d(g) for _, g in ents])
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    axis = np.ascontiguousarray(axis, dtype=np.float64).reshape(-1, 3)
    poi = np.ascontiguousarray(poi, dtype=np.float64)
    n = pos.shape[0]
    n_traj = n // per
    o = np.zeros(n); g = np.zeros(n); c = np.zeros(n_traj)
    st = lib().orc_info_cost(len(ents), _p(sizes, C.c_int32), xs, gs, _d(pos), _d(axis), n_traj, per, _d(poi),
                             float(cos_cut), float(w_i), float(eps), float(power_p), float(zero_eps),
                             int(bool(normalize)), _d(o), _d(g), _d(c))
    if st:
        raise OracleError(st, "info_cost")
    return o, g, c


def quantize_prob(p, observed, t_occ=0.5, t_free=0.5):
    """(codes, levels) of the per-voxel-probability map (S:69 states, P -> level = rne(63 P))."""
    p = np.ascontiguousarray(p, dtype=np.float32)
    obs = np.ascontiguousarray(observed, dtype=np.uint8)
    codes = np.zeros(p.shape, np.uint8); levels = np.zeros(p.shape, np.uint8)
    lib().orc_quantize_prob(_p(p, C.c_float), _p(obs, C.c_uint8), p.size, float(t_occ), float(t_free),
                            _p(codes, C.c_uint8), _p(levels, C.c_uint8))
    return codes, levels


# ------------------------------------------------------------ map integration (f3)

INTEGRATE_DEFAULTS = dict(p_hit=0.7, p_miss=0.4, p_min=0.12, p_max=0.97, max_range=5.0)


def voxel_filter(points, leaf):
    """(centroids [m, 3], counts [m]) of the voxel filter (reading Q33)."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    out = np.zeros((max(n, 1), 3)); cnt = np.zeros(max(n, 1), np.int32)
    m = C.c_int64()
    st = lib().orc_voxel_filter(_d(pts), n, float(leaf), _d(out), _p(cnt, C.c_int32), C.byref(m))
    if st:
        raise OracleError(st, "voxel_filter")
    return out[:m.value].copy(), cnt[:m.value].copy()


def new_logodds(shape_zyx):
    """A log-odds store with every voxel unobserved (NaN), indexed [z, y, x]."""
    return np.full(shape_zyx, np.nan, dtype=np.float32)


def integrate(L, voxel_size, map_origin, origin, points, leaf=0.0, p_hit=0.7, p_miss=0.4, p_min=0.12, p_max=0.97,
              max_range=5.0):
    """Integrate one cloud into the float32 log-odds store L ([z, y, x], in place, Q33-Q37).

    Returns (touched [z, y, x] uint8: 0 / 1 miss / 3 hit, number of rays)."""
    assert L.dtype == np.float32 and L.flags.c_contiguous
    nz, ny, nx = L.shape
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    mo = np.ascontiguousarray(map_origin, dtype=np.float64)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    touched = np.zeros(L.shape, np.uint8)
    nr = C.c_int64()
    st = lib().orc_integrate(_p(L, C.c_float), nx, ny, nz, float(voxel_size), _d(mo), _d(o), _d(pts), pts.shape[0],
                             float(p_hit), float(p_miss), float(p_min), float(p_max), float(max_range), float(leaf),
                             _p(touched, C.c_uint8), C.byref(nr))
    if st:
        raise OracleError(st, "integrate")
    return touched, nr.value


def occ_classify(L, t_occ=0.5, t_free=0.5):
    """(codes, levels) of a log-odds store (reading Q37)."""
    L = np.ascontiguousarray(L, dtype=np.float32)
    codes = np.zeros(L.shape, np.uint8); levels = np.zeros(L.shape, np.uint8)
    lib().orc_occ_classify(_p(L, C.c_float), L.size, float(t_occ), float(t_free), _p(codes, C.c_uint8),
                           _p(levels, C.c_uint8))
    return codes, levels
