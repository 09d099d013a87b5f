"""Python binding of libnbt (include/nbt.h): argument marshalling only.

Every step of the Information Distribution runs in libnbt's CUDA kernels; this module
converts numpy arrays / torch tensors to pointers, calls the C ABI function of the same
name and turns status codes into exceptions.  There is no CPU fallback: if libnbt.so is
missing, or no CUDA device is present, calls raise.

    import paper_2503_22588_b200 as nbt
    ctx = nbt.Ctx(0)
    m = nbt.Map(ctx, nbt.map_desc(256, 256, 256, 0.01)); m.upload(codes)
    cam = nbt.camera_from_fov(fov_h, fov_v, 64, 48)
    cloud = nbt.id_compute(ctx, m, poi, persp, cam, 1.5)    # -> IgCloud(xyz, gain, counts)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NBT_LIB") or os.path.join(_HERE, "libnbt.so")   # NBT_LIB: experiment builds

OK, ERR_INVALID_ARG, ERR_DEGENERATE, ERR_EMPTY, ERR_OUT_OF_MEMORY, ERR_CUDA, ERR_NCCL, ERR_STATE = range(8)
UNKNOWN, FREE, OCCUPIED = 0, 1, 2
OUTSIDE_UNKNOWN, OUTSIDE_CLIP = 0, 1
LAYOUT_LINEAR, LAYOUT_MORTON = 0, 1
(OPT_TRACE_REFILL_MIN, OPT_TRACE_CHUNK_MIN, OPT_TRACE_CARVEOUT, OPT_DELTA_SORT, OPT_FILTER_SORT, OPT_H2D_MODE,
 OPT_COPY_THREADS, OPT_WALK_WIDTH, OPT_VERBOSE) = range(1, 10)
SAMPLE_BALL, SAMPLE_SURFACE = 0, 1
(KERNEL_TRACE, KERNEL_FRAMES, KERNEL_FINALIZE, KERNEL_IDW, KERNEL_SAMPLE, KERNEL_MAP_UPDATE,
 KERNEL_INTEGRATE) = range(7)

# Every symbol include/nbt.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "nbt_abi_version", "nbt_status_string", "nbt_last_error_message",
    "nbt_ctx_create", "nbt_ctx_set_stream", "nbt_ctx_sync", "nbt_ctx_destroy", "nbt_ctx_launch_count",
    "nbt_ctx_set_option", "nbt_ctx_get_option",
    "nbt_ctx_set_profiling", "nbt_ctx_set_profiling_mask", "nbt_ctx_profile_read",
    "nbt_ctx_capture_begin", "nbt_ctx_capture_end", "nbt_graph_launch", "nbt_graph_profile_read", "nbt_graph_destroy",
    "nbt_map_desc_default", "nbt_map_create", "nbt_map_create_prob", "nbt_map_upload", "nbt_map_upload_prob",
    "nbt_map_update", "nbt_map_update_prob", "nbt_map_device_buffer", "nbt_map_download", "nbt_map_download_levels",
    "nbt_map_get_desc", "nbt_map_destroy",
    "nbt_camera_from_fov", "nbt_camera_from_grid_scaling", "nbt_camera_num_rays",
    "nbt_sample_perspectives", "nbt_id_compute", "nbt_id_compute_slice", "nbt_id_compute_rays", "nbt_id_finalize",
    "nbt_gather_create", "nbt_gather_export", "nbt_gather_attach", "nbt_gather_rows", "nbt_id_compute_gather",
    "nbt_gather_destroy", "nbt_gather_zero", "nbt_id_compute_rays_gather",
    "nbt_idbuf_create", "nbt_idbuf_push", "nbt_idbuf_clear", "nbt_idbuf_size", "nbt_ig_query", "nbt_ig_query_knn", "nbt_idbuf_destroy",
    "nbt_info_cost",
    "nbt_integrate_params_default", "nbt_occ_create", "nbt_occ_upload", "nbt_occ_download", "nbt_occ_integrate",
    "nbt_occ_stats", "nbt_occ_deltas", "nbt_occ_destroy", "nbt_voxel_filter",
    "nbt_debug_trace", "nbt_debug_frames", "nbt_debug_id_rays",
]


class NbtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class MapDesc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("voxel_size", C.c_double),
                ("origin", C.c_double * 3), ("gain", C.c_double * 3), ("outside_policy", C.c_int32),
                ("layout", C.c_int32), ("state_bits", C.c_int32)]


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("add_corners", C.c_int32),
                ("tan_half_fov_h", C.c_double), ("tan_half_fov_v", C.c_double)]

    @property
    def num_rays(self):
        return self.width * self.height + (4 if self.add_corners else 0)


class IntegrateParams(C.Structure):
    _fields_ = [("p_hit", C.c_double), ("p_miss", C.c_double), ("p_min", C.c_double), ("p_max", C.c_double),
                ("t_occ", C.c_double), ("t_free", C.c_double), ("max_range", C.c_double), ("leaf", C.c_double)]


class IgCloudC(C.Structure):
    _fields_ = [("xyz", C.c_void_p), ("gain", C.c_void_p), ("counts", C.c_void_p), ("on_device", C.c_int32)]


_lib = None


def lib():
    """Load libnbt.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libnbt.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, dbl, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
    sz = C.c_size_t
    sig = {
        "nbt_abi_version": ([], C.c_int),
        "nbt_status_string": ([C.c_int], C.c_char_p),
        "nbt_last_error_message": ([], C.c_char_p),
        "nbt_ctx_create": ([C.c_int, vp, C.POINTER(vp)], C.c_int),
        "nbt_ctx_set_stream": ([vp, vp], C.c_int),
        "nbt_ctx_sync": ([vp], C.c_int),
        "nbt_ctx_destroy": ([vp], None),
        "nbt_ctx_launch_count": ([vp], u64),
        "nbt_ctx_set_option": ([vp, i32, i64], C.c_int),
        "nbt_ctx_get_option": ([vp, i32, C.POINTER(i64)], C.c_int),
        "nbt_ctx_set_profiling": ([vp, C.c_int], C.c_int),
        "nbt_ctx_set_profiling_mask": ([vp, C.c_uint32], C.c_int),
        "nbt_ctx_profile_read": ([vp, i32, C.POINTER(C.c_double), C.POINTER(u64), C.c_int], C.c_int),
        "nbt_ctx_capture_begin": ([vp], C.c_int),
        "nbt_ctx_capture_end": ([vp, C.POINTER(vp)], C.c_int),
        "nbt_graph_launch": ([vp], C.c_int),
        "nbt_graph_profile_read": ([vp, i32, C.POINTER(C.c_double), C.POINTER(u64)], C.c_int),
        "nbt_graph_destroy": ([vp], None),
        "nbt_map_desc_default": ([C.POINTER(MapDesc), i32, i32, i32, dbl], None),
        "nbt_map_create": ([vp, C.POINTER(MapDesc), C.POINTER(vp)], C.c_int),
        "nbt_map_create_prob": ([vp, C.POINTER(MapDesc), C.POINTER(vp)], C.c_int),
        "nbt_map_update_prob": ([vp, vp, vp, vp, sz, C.c_int, dbl, dbl], C.c_int),
        "nbt_map_download_levels": ([vp, vp, sz], C.c_int),
        "nbt_map_upload": ([vp, vp, sz, C.c_int], C.c_int),
        "nbt_map_upload_prob": ([vp, vp, vp, sz, C.c_int, dbl, dbl], C.c_int),
        "nbt_map_update": ([vp, vp, vp, sz, C.c_int], C.c_int),
        "nbt_map_device_buffer": ([vp, C.POINTER(vp), C.POINTER(sz)], C.c_int),
        "nbt_map_download": ([vp, vp, sz], C.c_int),
        "nbt_map_get_desc": ([vp, C.POINTER(MapDesc)], C.c_int),
        "nbt_map_destroy": ([vp], None),
        "nbt_camera_from_fov": ([dbl, dbl, i32, i32, C.POINTER(Camera)], C.c_int),
        "nbt_camera_from_grid_scaling": ([dbl, dbl, dbl, dbl, dbl, C.POINTER(Camera)], C.c_int),
        "nbt_camera_num_rays": ([C.POINTER(Camera)], i32),
        "nbt_sample_perspectives": ([vp, vp, dbl, i32, u64, i32, vp, C.c_int], C.c_int),
        "nbt_id_compute": ([vp, vp, vp, vp, i32, C.c_int, C.POINTER(Camera), dbl, C.POINTER(IgCloudC)], C.c_int),
        "nbt_id_compute_slice": ([vp, vp, vp, vp, i32, C.c_int, i32, i32, C.POINTER(Camera), dbl,
                                  C.POINTER(IgCloudC)], C.c_int),
        "nbt_id_compute_rays": ([vp, vp, vp, vp, i32, C.c_int, i32, i32, C.POINTER(Camera), dbl, vp], C.c_int),
        "nbt_id_finalize": ([vp, vp, vp, vp, i32, C.c_int, C.POINTER(Camera), dbl, vp, C.POINTER(IgCloudC)],
                            C.c_int),
        "nbt_gather_create": ([vp, i32, i32, i32, C.POINTER(vp)], C.c_int),
        "nbt_gather_export": ([vp, vp], C.c_int),
        "nbt_gather_attach": ([vp, i32, vp], C.c_int),
        "nbt_gather_rows": ([vp, C.POINTER(IgCloudC)], C.c_int),
        "nbt_id_compute_gather": ([vp, vp, vp, vp, i32, C.c_int, i32, i32, i32, C.POINTER(Camera), dbl, vp],
                                  C.c_int),
        "nbt_gather_destroy": ([vp], None),
        "nbt_gather_zero": ([vp], C.c_int),
        "nbt_id_compute_rays_gather": ([vp, vp, vp, vp, i32, C.c_int, C.POINTER(Camera), dbl, vp], C.c_int),
        "nbt_idbuf_create": ([vp, i32, i32, C.POINTER(vp)], C.c_int),
        "nbt_idbuf_push": ([vp, C.POINTER(IgCloudC), i32], C.c_int),
        "nbt_idbuf_clear": ([vp], C.c_int),
        "nbt_idbuf_size": ([vp], i32),
        "nbt_ig_query": ([vp, vp, i32, C.c_int, dbl, dbl, i32, vp, C.c_int], C.c_int),
        "nbt_ig_query_knn": ([vp, vp, i32, C.c_int, dbl, dbl, i32, i32, vp, C.c_int], C.c_int),
        "nbt_idbuf_destroy": ([vp], None),
        "nbt_info_cost": ([vp, vp, vp, i32, i32, C.c_int, vp, dbl, dbl, dbl, dbl, dbl, i32, vp, vp, vp, C.c_int],
                          C.c_int),
        "nbt_integrate_params_default": ([C.POINTER(IntegrateParams), dbl], None),
        "nbt_occ_create": ([vp, C.POINTER(MapDesc), C.POINTER(vp)], C.c_int),
        "nbt_occ_upload": ([vp, vp, sz, C.c_int], C.c_int),
        "nbt_occ_download": ([vp, vp, sz], C.c_int),
        "nbt_occ_integrate": ([vp, vp, vp, vp, i64, C.c_int, C.POINTER(IntegrateParams)], C.c_int),
        "nbt_occ_stats": ([vp, C.POINTER(i64)], C.c_int),
        "nbt_occ_deltas": ([vp, vp, vp, vp, sz, C.POINTER(sz)], C.c_int),
        "nbt_occ_destroy": ([vp], None),
        "nbt_voxel_filter": ([vp, vp, i64, C.c_int, dbl, vp, vp, C.POINTER(i64)], C.c_int),
        "nbt_debug_trace": ([vp, vp, vp, vp, i32, i32, vp, vp, vp, vp], C.c_int),
        "nbt_debug_frames": ([vp, vp, vp, vp, i32, C.POINTER(Camera), dbl, vp, vp], C.c_int),
        "nbt_debug_id_rays": ([vp, vp, vp, vp, i32, C.POINTER(Camera), dbl, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("NBT_LIB") and not hasattr(L, name):
            continue                  # an older experiment build: only the calls it has
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _status_name(s):
    try:
        return lib().nbt_status_string(int(s)).decode()
    except Exception:  # noqa: BLE001 -- only used to format an error
        return f"status {s}"


def check(status):
    if status != OK:
        raise NbtError(status, lib().nbt_last_error_message().decode())


# ------------------------------------------------------------------ marshalling

def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x, dtype):
    """(pointer, on_device, keepalive) for a numpy array or torch tensor of `dtype`."""
    if x is None:
        return None, 0, None
    if _is_torch(x):
        import torch
        tdt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32,
               np.uint8: torch.uint8, np.uint64: torch.int64}[dtype]
        if x.dtype != tdt or not x.is_contiguous():
            raise TypeError(f"expected a contiguous {tdt} tensor")
        return C.c_void_p(x.data_ptr()), int(x.is_cuda), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return C.c_void_p(a.ctypes.data), 0, a


def _count(keep) -> int:
    """Number of elements of the array / tensor _ptr returned (0 for None)."""
    if keep is None:
        return 0
    return int(keep.numel()) if _is_torch(keep) else int(keep.size)


def _poi(poi):
    a = np.ascontiguousarray(poi, dtype=np.float64).reshape(3)
    return C.c_void_p(a.ctypes.data), a


# ------------------------------------------------------------------------ API

def nbt_abi_version():
    return lib().nbt_abi_version()


class Ctx:
    """nbt_ctx: one CUDA device + stream (a borrowed torch stream, or an owned one)."""

    def __init__(self, device=0, stream=None):
        h = C.c_void_p()
        s = C.c_void_p(int(stream)) if stream is not None else None
        check(lib().nbt_ctx_create(int(device), s, C.byref(h)))
        self.h = h
        self.device = device

    def set_stream(self, stream):
        check(lib().nbt_ctx_set_stream(self.h, C.c_void_p(int(stream)) if stream is not None else None))

    def sync(self):
        check(lib().nbt_ctx_sync(self.h))

    @property
    def launches(self):
        return int(lib().nbt_ctx_launch_count(self.h))

    def set_option(self, option, value):
        """nbt_ctx_set_option: a tuning option (OPT_*); no option changes any result."""
        check(lib().nbt_ctx_set_option(self.h, int(option), int(value)))

    def get_option(self, option):
        v = C.c_int64()
        check(lib().nbt_ctx_get_option(self.h, int(option), C.byref(v)))
        return int(v.value)

    def set_profiling_mask(self, kernels):
        """Record only these kernel families (iterable of KERNEL_* ids; empty = off)."""
        mask = 0
        for k in kernels:
            mask |= 1 << int(k)
        check(lib().nbt_ctx_set_profiling_mask(self.h, mask))

    def set_profiling(self, on=True):
        check(lib().nbt_ctx_set_profiling(self.h, int(bool(on))))

    def profile_read(self, kernel, reset=True):
        """(total_ms, launches) of a kernel family since the last reset (syncs the stream)."""
        ms, n = C.c_double(), C.c_uint64()
        check(lib().nbt_ctx_profile_read(self.h, int(kernel), C.byref(ms), C.byref(n), int(bool(reset))))
        return ms.value, int(n.value)

    def capture_begin(self):
        """Start recording the following calls on this ctx into a CUDA graph (device buffers only)."""
        check(lib().nbt_ctx_capture_begin(self.h))

    def capture_end(self):
        g = C.c_void_p()
        check(lib().nbt_ctx_capture_end(self.h, C.byref(g)))
        return Graph(g, self)

    def close(self):
        if getattr(self, "h", None):
            lib().nbt_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class Graph:
    """nbt_graph: a captured sequence of libnbt calls, replayed with one launch."""

    def __init__(self, h, ctx):
        self.h, self.ctx = h, ctx

    def launch(self):
        check(lib().nbt_graph_launch(self.h))

    def profile_read(self, kernel):
        ms, n = C.c_double(), C.c_uint64()
        check(lib().nbt_graph_profile_read(self.h, int(kernel), C.byref(ms), C.byref(n)))
        return ms.value, int(n.value)

    def close(self):
        if getattr(self, "h", None):
            lib().nbt_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def map_desc(nx, ny, nz, voxel_size, origin=(0.0, 0.0, 0.0), gain=None, outside_policy=OUTSIDE_UNKNOWN,
             layout=LAYOUT_LINEAR, state_bits=2):
    """nbt_map_desc: grid, voxel size, origin, Eq. 2 gains, outside policy, store layout
    (LAYOUT_LINEAR / LAYOUT_MORTON, or "linear" / "morton") and bits per voxel (2 or 8)."""
    d = MapDesc()
    lib().nbt_map_desc_default(C.byref(d), int(nx), int(ny), int(nz), float(voxel_size))
    d.origin[:] = [float(v) for v in origin]
    if gain is not None:
        d.gain[:] = [float(v) for v in gain]
    d.outside_policy = int(outside_policy)
    if isinstance(layout, str):
        layout = {"linear": LAYOUT_LINEAR, "morton": LAYOUT_MORTON}[layout]
    d.layout = int(layout)
    d.state_bits = int(state_bits)
    return d


class Map:
    """nbt_map: the device-resident 2-bit voxel store (row a1)."""

    def __init__(self, ctx: Ctx, desc: MapDesc, prob: bool = False):
        """prob=True: also store per-voxel probabilities for the exact Eq. 2 (f1)."""
        h = C.c_void_p()
        create = lib().nbt_map_create_prob if prob else lib().nbt_map_create
        check(create(ctx.h, C.byref(desc), C.byref(h)))
        self.h, self.ctx, self.desc, self.prob = h, ctx, desc, prob

    @property
    def shape(self):
        return (self.desc.nz, self.desc.ny, self.desc.nx)

    @property
    def nvox(self):
        return self.desc.nx * self.desc.ny * self.desc.nz

    def upload(self, codes):
        p, dev, keep = _ptr(codes, np.uint8)
        check(lib().nbt_map_upload(self.h, p, _count(keep), dev))      # the C side checks n == nx*ny*nz

    def upload_prob(self, p, observed, t_occ=0.5, t_free=0.5):
        pp, dev, k1 = _ptr(p, np.float32)
        po, dev2, k2 = _ptr(observed, np.uint8)
        if dev != dev2:
            raise ValueError("p and observed must both be host or both device")
        if _count(k1) != _count(k2):
            raise ValueError("p and observed differ in size")
        check(lib().nbt_map_upload_prob(self.h, pp, po, _count(k1), dev, float(t_occ), float(t_free)))

    def update(self, ijk, codes):
        pi, dev, k1 = _ptr(ijk, np.int32)
        pc, dev2, k2 = _ptr(codes, np.uint8)
        if dev != dev2:
            raise ValueError("ijk and codes must both be host or both device")
        n = _count(k2)
        if _count(k1) != 3 * n:
            raise ValueError("ijk must hold 3 ints per delta")
        check(lib().nbt_map_update(self.h, pi, pc, n, dev))

    def update_prob(self, ijk, p, observed, t_occ=0.5, t_free=0.5):
        pi, dev, k1 = _ptr(ijk, np.int32)
        pp, dev2, k2 = _ptr(p, np.float32)
        po, dev3, k3 = _ptr(observed, np.uint8)
        if not dev == dev2 == dev3:
            raise ValueError("ijk, p and observed must all be host or all device")
        n = _count(k2)
        if _count(k1) != 3 * n or _count(k3) != n:
            raise ValueError("ijk (3 per delta), p and observed differ in size")
        check(lib().nbt_map_update_prob(self.h, pi, pp, po, n, dev, float(t_occ), float(t_free)))

    def download_levels(self):
        out = np.empty(self.shape, np.uint8)
        check(lib().nbt_map_download_levels(self.h, C.c_void_p(out.ctypes.data), self.nvox))
        return out

    def device_buffer(self):
        p, n = C.c_void_p(), C.c_size_t()
        check(lib().nbt_map_device_buffer(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def download(self):
        out = np.empty(self.shape, np.uint8)
        check(lib().nbt_map_download(self.h, C.c_void_p(out.ctypes.data), self.nvox))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().nbt_map_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


# ------------------------------------------------------- map integration (row f3)

def integrate_params(voxel_size, **kw) -> IntegrateParams:
    """nbt_integrate_params with the defaults of nbt_integrate_params_default, overridden by kw."""
    prm = IntegrateParams()
    lib().nbt_integrate_params_default(C.byref(prm), float(voxel_size))
    for k, v in kw.items():
        setattr(prm, k, float(v))
    return prm


class OccMap:
    """nbt_occ: the float32 log-odds occupancy store that depth frames are integrated into."""

    def __init__(self, ctx: Ctx, desc: MapDesc):
        h = C.c_void_p()
        check(lib().nbt_occ_create(ctx.h, C.byref(desc), C.byref(h)))
        self.h, self.ctx, self.desc = h, ctx, desc

    @property
    def shape(self):
        return (self.desc.nz, self.desc.ny, self.desc.nx)

    @property
    def nvox(self):
        return self.desc.nx * self.desc.ny * self.desc.nz

    def upload(self, logodds):
        p, dev, keep = _ptr(logodds, np.float32)
        check(lib().nbt_occ_upload(self.h, p, _count(keep), dev))

    def download(self):
        out = np.empty(self.shape, np.float32)
        check(lib().nbt_occ_download(self.h, C.c_void_p(out.ctypes.data), self.nvox))
        return out

    def integrate(self, sensor, points, map: Map | None = None, params: IntegrateParams | None = None):
        """Integrate one cloud ([n, 3] float64, host array or CUDA tensor); stream-ordered."""
        ps, keep_s = _poi(sensor)
        pp, dev, keep = _ptr(points, np.float64)
        n = (keep.numel() // 3 if _is_torch(keep) else keep.size // 3) if keep is not None else 0
        prm = params if params is not None else integrate_params(self.desc.voxel_size)
        check(lib().nbt_occ_integrate(self.h, map.h if map is not None else None, ps, pp, n, dev, C.byref(prm)))

    def stats(self):
        """(points, rays after the filter, voxels updated, deltas) of the last integrate; syncs."""
        out = (C.c_int64 * 4)()
        check(lib().nbt_occ_stats(self.h, out))
        return tuple(int(v) for v in out)

    def deltas(self):
        """(ijk [k, 3] int32, codes [k], levels [k]) of the last integrate, unspecified order."""
        n = C.c_size_t()
        check(lib().nbt_occ_deltas(self.h, None, None, None, 0, C.byref(n)))
        k = n.value
        ijk = np.zeros((max(k, 1), 3), np.int32); codes = np.zeros(max(k, 1), np.uint8)
        levels = np.zeros(max(k, 1), np.uint8)
        check(lib().nbt_occ_deltas(self.h, C.c_void_p(ijk.ctypes.data), C.c_void_p(codes.ctypes.data),
                                   C.c_void_p(levels.ctypes.data), k, C.byref(n)))
        return ijk[:k], codes[:k], levels[:k]

    def close(self):
        if getattr(self, "h", None):
            lib().nbt_occ_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def voxel_filter(ctx: Ctx, points, leaf):
    """(centroids [m, 3], counts [m]) of the device voxel filter (cells in (iz, iy, ix) order)."""
    pp, dev, keep = _ptr(points, np.float64)
    n = (keep.numel() // 3 if _is_torch(keep) else keep.size // 3) if keep is not None else 0
    out = np.zeros((max(n, 1), 3)); cnt = np.zeros(max(n, 1), np.int32)
    m = C.c_int64()
    check(lib().nbt_voxel_filter(ctx.h, pp, n, dev, float(leaf), C.c_void_p(out.ctypes.data),
                                 C.c_void_p(cnt.ctypes.data), C.byref(m)))
    return out[:m.value].copy(), cnt[:m.value].copy()


def camera_from_fov(fov_h, fov_v, w, h) -> Camera:
    cam = Camera()
    check(lib().nbt_camera_from_fov(float(fov_h), float(fov_v), int(w), int(h), C.byref(cam)))
    return cam


def camera_from_grid_scaling(fov_h, fov_v, range_, voxel_size, s_g) -> Camera:
    cam = Camera()
    check(lib().nbt_camera_from_grid_scaling(float(fov_h), float(fov_v), float(range_), float(voxel_size),
                                             float(s_g), C.byref(cam)))
    return cam


def sample_perspectives(ctx: Ctx, poi, r_s, n, seed, mode=SAMPLE_BALL, out=None):
    """Eq. 1 on the device.  `out` may be a (n,3) float64 CUDA tensor; default: host numpy."""
    pp, keep = _poi(poi)
    if out is None:
        out = np.empty((n, 3), np.float64)
    po, dev, k = _ptr(out, np.float64)
    if _count(k) < 3 * int(n):
        raise ValueError("out holds fewer than 3 n values")
    check(lib().nbt_sample_perspectives(ctx.h, pp, float(r_s), int(n), int(seed) & (2 ** 64 - 1), int(mode), po, dev))
    return out


@dataclass
class IgCloud:
    xyz: object
    gain: object
    counts: object

    def as_c(self):
        px, dev, _ = _ptr(self.xyz, np.float64)
        pg, dev2, _ = _ptr(self.gain, np.float64)
        pc, dev3 = None, dev
        if self.counts is not None:
            pc, dev3, _ = _ptr(self.counts, np.uint64)
        if not dev == dev2 == dev3:
            raise ValueError("the cloud's buffers must all be host arrays or all CUDA tensors")
        return IgCloudC(px.value, pg.value, pc.value if pc is not None else None, dev)


def empty_cloud(n, device=None, counts=True):
    if device is None:
        return IgCloud(np.empty((n, 3)), np.empty(n), np.empty((n, 4), np.uint64) if counts else None)
    import torch
    return IgCloud(torch.empty((n, 3), dtype=torch.float64, device=device),
                   torch.empty(n, dtype=torch.float64, device=device),
                   torch.empty((n, 4), dtype=torch.int64, device=device) if counts else None)


def _check_cloud(cloud, n):
    """The caller-owned output buffers of a cloud hold at least n rows."""
    need = (("xyz", 3 * n), ("gain", n), ("counts", 4 * n))
    for name, k in need:
        buf = getattr(cloud, name)
        if buf is None:
            if name == "counts":
                continue
            raise ValueError(f"cloud.{name} is missing")
        if _count(buf) < k:
            raise ValueError(f"cloud.{name} holds {_count(buf)} values, {k} needed")


def nbt_id_compute(ctx: Ctx, m: Map, poi, persp, cam: Camera, range_, out: IgCloud | None = None,
                   first=0, stride=1):
    """The ID (rows a4-a8).  persp: (n,3) float64 numpy (host) or CUDA tensor.  With first/stride
    only rows first + i*stride are computed and written compactly (multi-GPU shards)."""
    pp, keep = _poi(poi)
    pper, dev, kp = _ptr(persp, np.float64)
    if _count(kp) % 3:
        raise ValueError("perspectives must be (n, 3) float64")
    n_src = _count(kp) // 3
    n = max(0, (n_src - first + stride - 1) // stride) if first < n_src else 0
    if out is None:
        out = empty_cloud(n)
    _check_cloud(out, n)
    oc = out.as_c()
    if (first, stride) == (0, 1):
        check(lib().nbt_id_compute(ctx.h, m.h, pp, pper, int(n_src), dev, C.byref(cam), float(range_), C.byref(oc)))
    else:
        check(lib().nbt_id_compute_slice(ctx.h, m.h, pp, pper, int(n_src), dev, int(first), int(stride),
                                         C.byref(cam), float(range_), C.byref(oc)))
    return out


id_compute = nbt_id_compute

ID_TOTALS = 5   # NBT_ID_TOTALS: T_U, T_F, T_O, L, T_G per perspective


def _device_totals(t, n):
    import torch
    if not (_is_torch(t) and t.is_cuda and t.dtype == torch.int64 and t.is_contiguous()):
        raise TypeError("totals must be a contiguous int64 CUDA tensor (the uint64 bits)")
    if t.numel() < ID_TOTALS * n:
        raise ValueError(f"totals holds {t.numel()} values, {ID_TOTALS * n} needed")
    return C.c_void_p(t.data_ptr())


def nbt_id_compute_rays(ctx: Ctx, m: Map, poi, persp, cam: Camera, range_, ray_rank, ray_world, out=None):
    """Ray shard ray_rank of ray_world of the ID (SURVEY 8(e) ray split): the (n, 5) int64 CUDA
    tensor of this shard's integer totals (T_U, T_F, T_O, L, T_G); sum over the shards
    (all-reduce), then nbt_id_finalize."""
    import torch
    pp, keep = _poi(poi)
    pper, dev, kp = _ptr(persp, np.float64)
    if _count(kp) % 3:
        raise ValueError("perspectives must be (n, 3) float64")
    n = _count(kp) // 3
    if out is None:
        out = torch.empty((n, ID_TOTALS), dtype=torch.int64, device=torch.device("cuda", ctx.device))
    pt = _device_totals(out, n)
    check(lib().nbt_id_compute_rays(ctx.h, m.h, pp, pper, int(n), dev, int(ray_rank), int(ray_world),
                                    C.byref(cam), float(range_), pt))
    return out


def nbt_id_finalize(ctx: Ctx, m: Map, poi, persp, cam: Camera, range_, totals, out: IgCloud | None = None):
    """The IG cloud of totals summed over every ray shard (bit-identical to nbt_id_compute)."""
    pp, keep = _poi(poi)
    pper, dev, kp = _ptr(persp, np.float64)
    if _count(kp) % 3:
        raise ValueError("perspectives must be (n, 3) float64")
    n = _count(kp) // 3
    pt = _device_totals(totals, n)
    if out is None:
        out = empty_cloud(n)
    _check_cloud(out, n)
    oc = out.as_c()
    check(lib().nbt_id_finalize(ctx.h, m.h, pp, pper, int(n), dev, C.byref(cam), float(range_), pt, C.byref(oc)))
    return out


id_compute_rays = nbt_id_compute_rays
id_finalize = nbt_id_finalize

PEER_HANDLE_BYTES = 64


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


class Gather:
    """Peer-memory gather buffer of the IG cloud (nbt_gather_*): this rank's rows of the whole
    cloud, filled by every rank's Gather.compute through CUDA IPC mappings."""

    def __init__(self, ctx: Ctx, rows: int, world: int, rank: int):
        h = C.c_void_p()
        check(lib().nbt_gather_create(ctx.h, int(rows), int(world), int(rank), C.byref(h)))
        self.h, self.ctx, self.rows, self.world, self.rank = h, ctx, int(rows), int(world), int(rank)

    def export(self) -> bytes:
        buf = (C.c_uint8 * PEER_HANDLE_BYTES)()
        check(lib().nbt_gather_export(self.h, buf))
        return bytes(buf)

    def attach(self, peer_rank: int, handle: bytes):
        buf = (C.c_uint8 * PEER_HANDLE_BYTES).from_buffer_copy(bytes(handle))
        check(lib().nbt_gather_attach(self.h, int(peer_rank), buf))

    def cloud(self) -> IgCloud:
        """This rank's whole cloud as CUDA tensors viewing the library's buffer."""
        import torch
        oc = IgCloudC()
        check(lib().nbt_gather_rows(self.h, C.byref(oc)))
        n = self.rows
        return IgCloud(torch.as_tensor(_DevArray(oc.xyz, (n, 3), "<f8"), device=f"cuda:{self.ctx.device}"),
                       torch.as_tensor(_DevArray(oc.gain, (n,), "<f8"), device=f"cuda:{self.ctx.device}"),
                       torch.as_tensor(_DevArray(oc.counts, (n, 4), "<i8"), device=f"cuda:{self.ctx.device}"))

    def compute(self, m: Map, poi, persp, cam: Camera, range_, first=None, stride=None, row0=0):
        """Perspectives first, first + stride, ... of `persp` (default: the strided shard
        rank, rank + world, ... of the whole set) into rows row0 + j of every rank's buffer."""
        pp, keep = _poi(poi)
        pper, dev, kp = _ptr(persp, np.float64)
        if _count(kp) % 3:
            raise ValueError("perspectives must be (n, 3) float64")
        n = _count(kp) // 3
        first = self.rank if first is None else first
        stride = self.world if stride is None else stride
        check(lib().nbt_id_compute_gather(self.ctx.h, m.h, pp, pper, int(n), dev, int(first), int(stride),
                                          int(row0), C.byref(cam), float(range_), self.h))

    def zero(self):
        check(lib().nbt_gather_zero(self.h))

    def compute_rays(self, m: Map, poi, persp, cam: Camera, range_):
        """This rank's ray shard of every perspective, its counts added into every rank's buffer
        (read as (n, 5) uint64 totals; nbt_id_compute_rays_gather)."""
        pp, keep = _poi(poi)
        pper, dev, kp = _ptr(persp, np.float64)
        if _count(kp) % 3:
            raise ValueError("perspectives must be (n, 3) float64")
        check(lib().nbt_id_compute_rays_gather(self.ctx.h, m.h, pp, pper, _count(kp) // 3, dev, C.byref(cam),
                                               float(range_), self.h))

    def totals(self, n: int):
        """The buffer's first n rows of totals as an (n, 5) int64 CUDA tensor view."""
        import torch
        oc = IgCloudC()
        check(lib().nbt_gather_rows(self.h, C.byref(oc)))
        return torch.as_tensor(_DevArray(oc.xyz, (n, ID_TOTALS), "<i8"), device=f"cuda:{self.ctx.device}")

    def close(self):
        if self.h:
            lib().nbt_gather_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class IdBuffer:
    """nbt_idbuf: device ring buffer of the last N_B IG clouds + the IDW query (row a9)."""

    def __init__(self, ctx: Ctx, capacity_nb=10, max_persp=4096):
        h = C.c_void_p()
        check(lib().nbt_idbuf_create(ctx.h, int(capacity_nb), int(max_persp), C.byref(h)))
        self.h, self.ctx = h, ctx

    def push(self, cloud: IgCloud, n=None):
        n = n if n is not None else _count(cloud.gain)
        _check_cloud(IgCloud(cloud.xyz, cloud.gain, None), int(n))
        oc = cloud.as_c()
        check(lib().nbt_idbuf_push(self.h, C.byref(oc), int(n)))

    def clear(self):
        check(lib().nbt_idbuf_clear(self.h))

    def __len__(self):
        return int(lib().nbt_idbuf_size(self.h))

    def query(self, xyz, power_p=2.0, zero_eps=1e-9, normalize=False, out=None, knn=0):
        """Eq. 4 at (n, 3) positions; knn > 0: only the knn nearest perspectives of each entry (Q22)."""
        pq, qdev, kq = _ptr(xyz, np.float64)
        if _count(kq) % 3:
            raise ValueError("queries must be (n, 3) float64")
        nq = _count(kq) // 3
        if out is None:
            out = np.empty(nq, np.float64)
        po, odev, ko = _ptr(out, np.float64)
        if _count(ko) < nq:
            raise ValueError("out holds fewer values than queries")
        check(lib().nbt_ig_query_knn(self.h, pq, int(nq), qdev, float(power_p), float(zero_eps),
                                     int(bool(normalize)), int(knn), po, odev))
        return out

    def info_cost(self, pos, axis, poses_per_traj, poi, cos_theta_cut, w_i, eps=1e-7, power_p=2.0, zero_eps=1e-9,
                  normalize=False, out=None):
        """f2: (O per pose, G per pose, c_I per trajectory) -- host numpy unless out=(o, g, c) tensors."""
        pp, pdev, kp = _ptr(pos, np.float64)
        pa, adev, ka = _ptr(axis, np.float64)
        if pdev != adev:
            raise ValueError("pos and axis must both be host or both device")
        if _count(kp) % 3 or _count(ka) != _count(kp):
            raise ValueError("pos and axis must both be (n, 3) float64")
        n = _count(kp) // 3
        n_traj = n // int(poses_per_traj)
        if out is None:
            out = (np.empty(n), np.empty(n), np.empty(n_traj))
        po, odev, k0 = _ptr(out[0], np.float64)
        pg, _, k1 = _ptr(out[1], np.float64)
        pc, _, k2 = _ptr(out[2], np.float64)
        if _count(k0) < n or _count(k1) < n or _count(k2) < n_traj:
            raise ValueError("out buffers too small")
        ppoi, keep = _poi(poi)
        check(lib().nbt_info_cost(self.h, pp, pa, int(n_traj), int(poses_per_traj), pdev, ppoi, float(cos_theta_cut),
                                  float(w_i), float(eps), float(power_p), float(zero_eps), int(bool(normalize)),
                                  po, pg, pc, odev))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().nbt_idbuf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def nbt_ig_query(buf: IdBuffer, xyz, power_p=2.0, zero_eps=1e-9, normalize=False, out=None):
    return buf.query(xyz, power_p, zero_eps, normalize, out)


def debug_trace(ctx: Ctx, m: Map, o_q16, e_q16, max_visits=1024):
    """Per-ray device walks of explicit Q16 segments: (ijk [n,max,3], codes [n,max], len [n], counts [n,4])."""
    o = np.ascontiguousarray(o_q16, dtype=np.int32).reshape(-1, 3)
    e = np.ascontiguousarray(e_q16, dtype=np.int32).reshape(-1, 3)
    if o.shape != e.shape:
        raise ValueError("o and e must hold the same number of segments")
    n = o.shape[0]
    ijk = np.zeros((n, max_visits, 3), np.int32)
    codes = np.zeros((n, max_visits), np.uint8)
    ln = np.zeros(n, np.int32)
    cnt = np.zeros((n, 4), np.uint32)
    check(lib().nbt_debug_trace(ctx.h, m.h, C.c_void_p(o.ctypes.data), C.c_void_p(e.ctypes.data), n, max_visits,
                                C.c_void_p(ijk.ctypes.data), C.c_void_p(codes.ctypes.data),
                                C.c_void_p(ln.ctypes.data), C.c_void_p(cnt.ctypes.data)))
    return ijk, codes, ln, cnt


def debug_id_rays(ctx: Ctx, m: Map, poi, persp, cam: Camera, range_):
    """Per-ray (n_U, n_F, n_O, lookups, stop) of the production trace kernel: [n, N_E, 5] uint32."""
    pp, keep = _poi(poi)
    P = np.ascontiguousarray(persp, dtype=np.float64).reshape(-1, 3)
    out = np.zeros((P.shape[0], cam.num_rays, 5), np.uint32)
    check(lib().nbt_debug_id_rays(ctx.h, m.h, pp, C.c_void_p(P.ctypes.data), P.shape[0], C.byref(cam),
                                  float(range_), C.c_void_p(out.ctypes.data)))
    return out


def debug_frames(ctx: Ctx, m: Map, poi, persp, cam: Camera, range_):
    pp, keep = _poi(poi)
    P = np.ascontiguousarray(persp, dtype=np.float64).reshape(-1, 3)
    q = np.zeros((P.shape[0], 18), np.int32)
    st = np.zeros(P.shape[0], np.int32)
    check(lib().nbt_debug_frames(ctx.h, m.h, pp, C.c_void_p(P.ctypes.data), P.shape[0], C.byref(cam),
                                 float(range_), C.c_void_p(q.ctypes.data), C.c_void_p(st.ctypes.data)))
    return q, st
