"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no sampling by Eq. 1, no frames,
no rays, no traversal, no scoring, no IDW).  It only produces the *inputs* the
paper's workloads would feed the Information Distribution (ID): three-state voxel
maps, the configuration table, IDW query positions and map-delta lists.  Both
sides (oracle/ and the CUDA path) consume exactly the same arrays.

Recipes (stated in DESIGN.md "Input recipe"):

* SYN(N, s, R_o, seed) -- the paper's "object inside a demonstrator" scene
   as a dense uint8 code grid, x fastest:
  background Free; occupied spherical shell R_o-2 <= r < R_o around the PoI;
  Unknown interior r < R_o-2; an occupied 2-voxel table slab 2 voxels below
  the object within 0.35 N of the centre (square); Unknown beyond 0.45 N from
  the map centre (unobserved space); an Unknown occlusion shadow behind the
  object as seen from a past camera c0 = PoI + (0, -0.4N, 0.2N); speckle:
  each remaining Free voxel becomes Unknown w.p. 0.02 or Occupied w.p. 5e-4.
* RAND(N, pU, pF, pO, seed) -- i.i.d. codes, for parity fuzzing.

Codes follow SURVEY.md section 8(a) row a1: 0 = Unknown, 1 = Free, 2 = Occupied.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

UNKNOWN, FREE, OCCUPIED = 0, 1, 2

# Azure-Kinect-like camera used by every config: FoV 75 x 65 degrees.
FOV_H = math.radians(75.0)
FOV_V = math.radians(65.0)


def poi_voxel_centre(n: int, voxel_size: float, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    """PoI at the centre of voxel (N/2, N/2, N/2) in world units."""
    c = (n // 2 + 0.5) * voxel_size
    return np.array([origin[0] + c, origin[1] + c, origin[2] + c], dtype=np.float64)


def syn_map(n: int, r_o: float, seed: int) -> np.ndarray:
    """SYN(N, s, R_o, seed): dense uint8 codes of shape (N, N, N) indexed [z, y, x].

    Distances are measured in voxel units between voxel centres; s only scales
    the world frame and does not change the codes.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    codes = np.empty((n, n, n), dtype=np.uint8)
    c = n // 2 + 0.5                       # PoI (voxel centre) in voxel units
    mc = n / 2.0                           # map centre
    ax = np.arange(n, dtype=np.float64) + 0.5
    X, Y = np.meshgrid(ax, ax, indexing="xy")          # [y, x]
    c0 = np.array([c, c - 0.4 * n, c + 0.2 * n])
    poi = np.array([c, c, c])
    v_poi = poi - c0
    d_poi2 = float(v_poi @ v_poi)
    table_top = c - r_o - 2.0              # slab occupies [table_top - 2, table_top)
    for k in range(n):
        z = k + 0.5
        sl = np.full((n, n), FREE, dtype=np.uint8)
        # occlusion shadow behind the object as seen from c0
        px, py, pz = X - c0[0], Y - c0[1], z - c0[2]
        dist = np.sqrt(px * px + py * py + pz * pz)
        with np.errstate(invalid="ignore", divide="ignore"):
            t_cl = (px * v_poi[0] + py * v_poi[1] + pz * v_poi[2]) / dist
        perp2 = d_poi2 - t_cl * t_cl
        r_poi2 = (X - c) ** 2 + (Y - c) ** 2 + (z - c) ** 2
        shadow = (t_cl > 0) & (t_cl < dist) & (perp2 < r_o * r_o) & (r_poi2 >= r_o * r_o)
        sl[shadow] = UNKNOWN
        # unobserved space far from the map centre
        r_mc2 = (X - mc) ** 2 + (Y - mc) ** 2 + (z - mc) ** 2
        sl[r_mc2 > (0.45 * n) ** 2] = UNKNOWN
        # table slab
        if table_top - 2.0 <= z < table_top:
            tab = (np.abs(X - mc) <= 0.35 * n) & (np.abs(Y - mc) <= 0.35 * n)
            sl[tab] = OCCUPIED
        # object: occupied shell, unknown interior
        sl[(r_poi2 < r_o * r_o) & (r_poi2 >= (r_o - 2.0) ** 2)] = OCCUPIED
        sl[r_poi2 < (r_o - 2.0) ** 2] = UNKNOWN
        codes[k] = sl
    # speckle on the remaining Free voxels (drawn for every voxel, in [z, y, x] order)
    flat = codes.reshape(-1)
    for start in range(0, flat.size, 1 << 24):
        u = rng.random(min(1 << 24, flat.size - start))
        seg = flat[start:start + u.size]
        free = seg == FREE
        seg[free & (u < 0.02)] = UNKNOWN
        seg[free & (u >= 0.02) & (u < 0.02 + 5e-4)] = OCCUPIED
    return codes


def rand_map(n, p_u=0.3, p_f=0.65, p_o=0.05, seed=0, shape=None) -> np.ndarray:
    """RAND(N, pU, pF, pO, seed): i.i.d. codes, shape (nz, ny, nx)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = shape or (n, n, n)
    u = rng.random(shape)
    out = np.full(shape, OCCUPIED, dtype=np.uint8)
    out[u < p_u + p_f] = FREE
    out[u < p_u] = UNKNOWN
    return out


Q16 = 65536   # ray-walk fixed point: 65536 units per voxel (reading Q19)


def random_segments_q16(count: int, lo: float, hi: float, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Random ray segments in Q16 voxel coordinates (int32), for DDA fuzzing."""
    rng = np.random.Generator(np.random.PCG64(seed))
    o = np.round(rng.uniform(lo, hi, (count, 3)) * Q16).astype(np.int32)
    e = np.round(rng.uniform(lo, hi, (count, 3)) * Q16).astype(np.int32)
    return o, e


def tie_segments_q16(count: int, n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Segments (Q16) whose endpoints sit on voxel faces / edges / corners (exact ties)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    o = rng.integers(0, n, (count, 3)) * Q16
    e = rng.integers(0, n, (count, 3)) * Q16
    half = rng.integers(0, 2, (count, 3)) * (Q16 // 2)
    o = o + half * rng.integers(0, 2, (count, 3))
    e = e + half * rng.integers(0, 2, (count, 3))
    return o.astype(np.int32), e.astype(np.int32)


def query_points(count: int, poi, r_s: float, lo: float, hi: float, seed: int) -> np.ndarray:
    """IDW query positions uniform in the shell lo*r_S..hi*r_S around the PoI (config E)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    d = rng.standard_normal((count, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = r_s * rng.uniform(lo, hi, count)
    return np.asarray(poi, dtype=np.float64)[None, :] + d * r[:, None]


def cycle_deltas(n: int, poi_vox, cycle: int, codes: np.ndarray, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Config E map deltas for one receding-horizon cycle.

    Carve a radius-6 ball Unknown->Free near the moving PoI; a 10x10x20 box moving
    2 voxels/cycle toggles Free<->Occupied; 500 random Free->Unknown.  Returns
    (ijk int32 [n,3], codes uint8 [n]) in application order.  `codes` (the map as
    currently known, [z,y,x]) is only read to pick the toggled value.
    """
    rng = np.random.Generator(np.random.PCG64(seed + 7919 * cycle))
    px, py, pz = (int(round(v)) for v in poi_vox)
    ijk, val = [], []
    r = np.arange(-6, 7)
    gz, gy, gx = np.meshgrid(r, r, r, indexing="ij")
    ball = (gx * gx + gy * gy + gz * gz) <= 36
    pts = np.stack([gx[ball] + px + 20, gy[ball] + py, gz[ball] + pz], axis=1)
    pts = pts[(pts >= 0).all(1) & (pts < n).all(1)]
    sel = codes[pts[:, 2], pts[:, 1], pts[:, 0]] == UNKNOWN
    ijk.append(pts[sel]); val.append(np.full(int(sel.sum()), FREE, np.uint8))
    bx0 = (2 * cycle) % max(1, n - 10)
    bx, by, bz = np.meshgrid(np.arange(bx0, bx0 + 10), np.arange(n // 4, n // 4 + 10),
                             np.arange(n // 2 - 10, n // 2 + 10), indexing="ij")
    box = np.stack([bx.ravel(), by.ravel(), bz.ravel()], axis=1)
    box = box[(box < n).all(1)]
    cur = codes[box[:, 2], box[:, 1], box[:, 0]]
    tog = np.where(cur == OCCUPIED, FREE, OCCUPIED).astype(np.uint8)
    keep = cur != UNKNOWN
    ijk.append(box[keep]); val.append(tog[keep])
    rnd = rng.integers(0, n, (500, 3))
    ijk.append(rnd); val.append(np.full(500, UNKNOWN, np.uint8))
    return np.concatenate(ijk).astype(np.int32), np.concatenate(val).astype(np.uint8)


@dataclass(frozen=True)
class Config:
    """One row of SURVEY.md 8(d): map, perspective set, ray lattice and range."""
    name: str
    n: int                   # map edge in voxels
    voxel_size: float        # s_Vox, world units
    r_o: float               # object radius (voxels) of SYN
    map_seed: int
    n_persp: int             # N_P
    persp_radius: float      # r_S (world units)
    persp_mode: int          # 0 = ball (Eq. 1), 1 = surface
    persp_seed: int
    width: int               # ray lattice W
    height: int              # ray lattice H
    range_: float            # d_Cam (world units)
    extra: dict = field(default_factory=dict)

    @property
    def poi(self) -> np.ndarray:
        return poi_voxel_centre(self.n, self.voxel_size)

    @property
    def rays_per_id(self) -> int:
        return self.n_persp * self.width * self.height

    def map_codes(self) -> np.ndarray:
        return syn_map(self.n, self.r_o, self.map_seed)


CONFIGS = {
    # configs[0] of BASELINE.json: the small case the oracle finishes in seconds
    "A": Config("A", 64, 1.0, 8.0, 0, 16, 24.0, 1, 0, 32, 24, 64.0),
    # configs[1]: 256^3, 1 cm voxels, 512 perspectives x 64x48 rays (the bench workload)
    "B": Config("B", 256, 0.01, 15.0, 1, 512, 1.0, 0, 1, 64, 48, 1.5),
    # configs[2]: 256 perspectives at full 640x480 sensor resolution
    "C": Config("C", 256, 0.01, 15.0, 1, 256, 1.0, 0, 2, 640, 480, 1.5),
    # north_star target: >= 512 perspectives x 640x480 on 256^3 within one 100 ms MHP cycle
    "C'": Config("C'", 256, 0.01, 15.0, 1, 512, 1.0, 0, 2, 640, 480, 1.5),
    # configs[3]: 512^3 map, 4096 perspectives x 160x120 rays (multi-GPU)
    "D": Config("D", 512, 0.01, 15.0, 3, 4096, 1.0, 0, 3, 160, 120, 3.86),
    # configs[4]: receding-horizon loop on B's map and camera
    "E": Config("E", 256, 0.01, 15.0, 1, 512, 1.0, 0, 1000, 64, 48, 1.5,
                extra={"cycles": 200, "n_b": 10, "queries": 1984, "power_p": 2.0}),
}


# ----------------------------------------------------------- sensor clouds

@dataclass(frozen=True)
class CloudConfig:
    """A map-integration workload (DESIGN.md input recipe, row f3): depth frames of the
    SYN scene taken from sensors circling the PoI, integrated into an empty map."""
    name: str
    n: int                   # map edge in voxels
    voxel_size: float        # s_Vox
    r_o: float               # object radius (voxels), as SYN
    width: int               # depth image W (Azure Kinect NFOV unbinned: 640 x 576)
    height: int
    sensor_dist: float       # sensor distance to the PoI (world units)
    n_clouds: int            # frames per workload (one per sensor pose)
    leaf: float              # voxel-filter leaf (world units)
    max_range: float         # integration range (world units)
    seed: int

    @property
    def poi(self) -> np.ndarray:
        return poi_voxel_centre(self.n, self.voxel_size)

    def sensor(self, k: int) -> np.ndarray:
        """Pose k: on a circle around the PoI, 25 degrees above its horizontal plane."""
        phi = 2.0 * math.pi * (k + 0.125) / max(1, self.n_clouds)
        el = math.radians(25.0)
        d = np.array([math.cos(phi) * math.cos(el), math.sin(phi) * math.cos(el), math.sin(el)])
        return self.poi + self.sensor_dist * d

    def cloud(self, k: int) -> np.ndarray:
        return sensor_cloud(self.n, self.voxel_size, self.r_o, self.sensor(k), self.poi, self.width, self.height,
                            seed=self.seed + 104729 * k)


def sensor_cloud(n: int, voxel_size: float, r_o: float, sensor, target, width: int, height: int,
                 noise: float = 1e-3, drop: float = 0.01, seed: int = 0) -> np.ndarray:
    """Synthetic depth frame of the SYN scene (world units, float64 [m, 3]).

    The scene is SYN's geometry as surfaces: the object sphere (radius r_o voxels at
    the PoI), the table top (the slab's upper face, a square of half-side 0.35 N about
    the map centre) and the boundary of observed space as a spherical wall of radius
    0.45 N about the map centre.  A pinhole sensor at `sensor` looks at `target`
    (up hint +z) over a width x height pixel lattice spanning the 75 x 65 degree FoV;
    each pixel returns the nearest surface along its ray, with N(0, noise) depth noise,
    and is dropped w.p. `drop` (invalid depth).  Scene generation only: none of the
    mapping method's arithmetic.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    s = voxel_size
    o = np.asarray(sensor, dtype=np.float64)
    tgt = np.asarray(target, dtype=np.float64)
    fwd = tgt - o
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 0.0, 1.0])
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    u = np.linspace(-1.0, 1.0, width) * math.tan(FOV_H / 2)
    v = np.linspace(-1.0, 1.0, height) * math.tan(FOV_V / 2)
    U, V = np.meshgrid(u, v, indexing="xy")
    d = fwd[None, :] + U.reshape(-1, 1) * right[None, :] + V.reshape(-1, 1) * up[None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    inf = np.full(d.shape[0], np.inf)
    # object sphere (outside surface)
    c = (n // 2 + 0.5) * s
    oc = o - np.array([c, c, c])
    b = d @ oc
    disc = b * b - (oc @ oc - (r_o * s) ** 2)
    t_obj = np.where(disc >= 0, -b - np.sqrt(np.maximum(disc, 0.0)), np.inf)
    t_obj = np.where(t_obj > 0, t_obj, np.inf)
    # table top plane
    mc = n / 2.0 * s
    z_top = (n // 2 + 0.5 - r_o - 2.0) * s
    with np.errstate(divide="ignore", invalid="ignore"):
        t_tab = (z_top - o[2]) / d[:, 2]
    hit = o[None, :] + t_tab[:, None] * d
    ok = (t_tab > 0) & (np.abs(hit[:, 0] - mc) <= 0.35 * n * s) & (np.abs(hit[:, 1] - mc) <= 0.35 * n * s)
    t_tab = np.where(ok, t_tab, inf)
    # boundary wall (inside surface of a sphere about the map centre)
    om = o - np.array([mc, mc, mc])
    b2 = d @ om
    disc2 = b2 * b2 - (om @ om - (0.45 * n * s) ** 2)
    t_wall = np.where(disc2 >= 0, -b2 + np.sqrt(np.maximum(disc2, 0.0)), np.inf)
    t = np.minimum(np.minimum(t_obj, t_tab), t_wall)
    t = t + rng.normal(0.0, noise, t.shape)
    keep = np.isfinite(t) & (t > 0) & (rng.random(t.shape) >= drop)
    return o[None, :] + t[keep, None] * d[keep]


CLOUD_CONFIGS = {
    # small: 64^3 map, 160 x 144 frames (oracle in well under a second)
    "F0": CloudConfig("F0", 64, 0.04, 4.0, 160, 144, 0.6, 4, 0.04, 1.2, 11),
    # full: config B's 256^3 / 1 cm map, Azure Kinect NFOV unbinned 640 x 576 frames
    "F": CloudConfig("F", 256, 0.01, 15.0, 640, 576, 0.6, 8, 0.01, 1.2, 12),
}
