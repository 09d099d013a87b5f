// The online local Information Distribution on the device.
//
//   k_persp_frames  per perspective: view frame (Q4) and its Q16 quantisation
//                   (Q19), bound checks; zeroes the per-perspective totals.
//   k_id_trace      persistent warps pull chunks of one perspective's rays; each lane
//                   builds its ray's endpoint on the far plane in registers (P:158-169,
//                   Q27), walks the exact integer 3D-DDA (Q13) through the 2-bit map,
//                   stops at the first Occupied voxel, and counts visits per
//                   state (Eq. 2 as integer counts, Q26).  Lanes that finish refill
//                   with their next ray, so the warp keeps stepping until the whole
//                   chunk is done.  One warp reduction + 4 u64 atomics per chunk.
//   k_id_finalize   g_P = ((T_U g_U + T_F g_F) + T_O g_O) / N_E  (Q26)
//
// The traversal is integer-only: voxel coordinates are Q16 fixed point (65536 per
// voxel).  The next boundary crossed is the axis minimising N_a/|D_a| (N_a = distance
// to its next boundary, D = E - O), compared exactly through the pairwise terms
// f_ab = N_a|D_b| - N_b|D_a| (int64) kept incrementally: a step along a adds
// 65536|D_b| to f_ab.  Exact ties are broken by (positive direction first, then axis
// order) through a -1 bias folded into f_ab at ray start, so each step is three sign
// tests and two 64-bit adds.
#include "nbt_internal.cuh"

namespace nbt {
namespace {

constexpr int kFrameInts = 20;   // O, A, Rh, Uh, Rc, Uc (3 each), status, pad
constexpr int kWarpsPerBlock = 8;

struct MapView {
    const uint32_t *__restrict__ words;
    int nx, ny, nz;
    int px;          // padded x extent
    int pxy;         // padded x*y extent
    int policy;      // NBT_OUTSIDE_UNKNOWN / NBT_OUTSIDE_CLIP
};

__device__ __forceinline__ uint32_t code_at(const MapView &m, uint32_t idx)
{
    uint32_t w = __ldg(m.words + (idx >> 4));
    return __funnelshift_r(w, 0u, idx << 1) & 3u;   // shift amount is taken mod 32
}

// Per-ray traversal state (all integer).
struct Ray {
    long long fxy, fxz, fyz;   // biased pairwise decision terms (negative -> first axis first)
    long long kx, ky, kz;      // 65536 * |D_a|
    uint32_t idx;              // padded linear voxel index (fast path)
    int dX, dY, dZ;            // idx increments of a step along x, y, z
    int s, n;                  // current step (0 = origin voxel), total steps
    int s0;                    // step at which the walk entered the grid
    uint32_t nf;               // Free voxels seen in the grid
    uint32_t pre;              // visits outside the grid before entering it
    int vx, vy, vz;            // voxel coordinates (slow path / debug only)
    int sx, sy, sz;            // +-1 per axis
};

__device__ __forceinline__ void ray_setup(Ray &r, const int o[3], const int e[3])
{
    int D[3], ad[3], neg[3], v[3], N[3];
    int n = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        D[a] = e[a] - o[a];                      // |D| < 2^31: both ends inside (-2^30, 2^30)
        neg[a] = D[a] < 0;
        ad[a] = neg[a] ? -D[a] : D[a];
        v[a] = o[a] >> 16;                       // floor
        int ve = e[a] >> 16;
        n += (ve > v[a]) ? ve - v[a] : v[a] - ve;
        N[a] = neg[a] ? o[a] - v[a] * 65536 : (v[a] + 1) * 65536 - o[a];   // in [0, 65536]
    }
    // tie favours the lower axis unless it moves negatively and the other positively
    long long exy = (long long)N[0] * ad[1] - (long long)N[1] * ad[0];
    long long exz = (long long)N[0] * ad[2] - (long long)N[2] * ad[0];
    long long eyz = (long long)N[1] * ad[2] - (long long)N[2] * ad[1];
    r.fxy = exy - ((neg[0] && !neg[1]) ? 0 : 1);
    r.fxz = exz - ((neg[0] && !neg[2]) ? 0 : 1);
    r.fyz = eyz - ((neg[1] && !neg[2]) ? 0 : 1);
    r.kx = (long long)ad[0] << 16;
    r.ky = (long long)ad[1] << 16;
    r.kz = (long long)ad[2] << 16;
    r.sx = neg[0] ? -1 : 1;
    r.sy = neg[1] ? -1 : 1;
    r.sz = neg[2] ? -1 : 1;
    r.vx = v[0]; r.vy = v[1]; r.vz = v[2];
    r.s = 0;
    r.n = n;
    r.nf = 0;
    r.pre = 0;
}

// Choose the next axis (0/1/2) and update the decision terms.
__device__ __forceinline__ int ray_advance(Ray &r)
{
    if (r.fxy < 0 && r.fxz < 0) {
        r.fxy += r.ky; r.fxz += r.kz;
        return 0;
    }
    if (r.fyz < 0) {
        r.fxy -= r.kx; r.fyz += r.kz;
        return 1;
    }
    r.fxz -= r.kx; r.fyz -= r.ky;
    return 2;
}

__device__ __forceinline__ bool inside(const MapView &m, int x, int y, int z)
{
    return (unsigned)x < (unsigned)m.nx && (unsigned)y < (unsigned)m.ny && (unsigned)z < (unsigned)m.nz;
}

// Origin outside the grid (rare): step with explicit bounds checks until the walk
// enters the grid or ends.  Returns true if the ray is finished.
template <bool RECORD>
__device__ bool ray_enter(Ray &r, const MapView &m, int32_t *rec_ijk, uint8_t *rec_code, int max_visits)
{
    while (!inside(m, r.vx, r.vy, r.vz)) {
        if (RECORD && r.s < max_visits) {
            rec_ijk[3 * r.s] = r.vx; rec_ijk[3 * r.s + 1] = r.vy; rec_ijk[3 * r.s + 2] = r.vz;
            rec_code[r.s] = 255;
        }
        r.pre++;
        if (r.s == r.n) return true;
        int a = ray_advance(r);
        if (a == 0) r.vx += r.sx; else if (a == 1) r.vy += r.sy; else r.vz += r.sz;
        r.s++;
    }
    r.s0 = r.s;
    r.idx = (uint32_t)(r.vx + 1) + (uint32_t)m.px * (uint32_t)(r.vy + 1) + (uint32_t)m.pxy * (uint32_t)(r.vz + 1);
    r.dX = r.sx;
    r.dY = r.sy * m.px;
    r.dZ = r.sz * m.pxy;
    return false;
}

struct Counts { uint32_t u, f, o, l; };

// Fast in-grid walk.  Ends on the first Occupied voxel, on leaving the grid (sentinel
// code 3, Q14 tail rule: the remaining n - s + 1 visits are all outside) or at the
// endpoint voxel.
template <bool RECORD>
__device__ void ray_walk(Ray &r, const MapView &m, Counts &c, int32_t *rec_ijk, uint8_t *rec_code, int max_visits)
{
    for (;;) {
        uint32_t code = code_at(m, r.idx);
        if (RECORD && r.s < max_visits) {
            rec_ijk[3 * r.s] = r.vx; rec_ijk[3 * r.s + 1] = r.vy; rec_ijk[3 * r.s + 2] = r.vz;
            rec_code[r.s] = code == 3 ? 255 : (uint8_t)code;
        }
        if (code >= 2u) {
            uint32_t tail = 0;
            uint32_t l;
            if (code == 2u) {
                l = r.s - r.s0 + 1;
                c.o += 1;
                c.u += l - r.nf - 1;
            } else {
                l = r.s - r.s0;
                tail = r.n - r.s + 1;
                c.u += l - r.nf;
                if (RECORD) {
                    for (int s = r.s + 1; s <= r.n && s < max_visits; ++s) {
                        int a = ray_advance(r);
                        if (a == 0) r.vx += r.sx; else if (a == 1) r.vy += r.sy; else r.vz += r.sz;
                        rec_ijk[3 * s] = r.vx; rec_ijk[3 * s + 1] = r.vy; rec_ijk[3 * s + 2] = r.vz;
                        rec_code[s] = 255;
                    }
                }
            }
            if (m.policy == NBT_OUTSIDE_UNKNOWN) c.u += r.pre + tail;
            c.f += r.nf;
            c.l += l;
            return;
        }
        r.nf += code;
        if (r.s == r.n) {
            uint32_t l = r.s - r.s0 + 1;
            c.u += l - r.nf + (m.policy == NBT_OUTSIDE_UNKNOWN ? r.pre : 0);
            c.f += r.nf;
            c.l += l;
            return;
        }
        int a = ray_advance(r);
        r.idx += (a == 0) ? r.dX : ((a == 1) ? r.dY : r.dZ);
        if (RECORD) { if (a == 0) r.vx += r.sx; else if (a == 1) r.vy += r.sy; else r.vz += r.sz; }
        r.s++;
    }
}

// ------------------------------------------------------------------ frames (a4)

__device__ __forceinline__ bool rne_q16(double v, int *out)
{
    double q = __dmul_rn(v, 65536.0);
    if (!(fabs(q) < 1073741824.0)) return false;
    *out = __double2int_rn(q);   // round half to even
    return true;
}

__device__ __forceinline__ double dot3_sq(double a, double b, double c)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c));
}

struct FrameArgs {
    const double *persp;
    int32_t first, stride, n;
    double poi[3];
    double origin[3];
    double voxel_size;
    double range;
    nbt_camera cam;
};

// Frame of perspective p: fwd = unit(PoI - p), right = unit(fwd x z) or
// unit(fwd x x) when |fwd x z| < 1e-6 (Q4), up = right x fwd; every product, sum
// and quotient rounded once (no FMA contraction) so the result is reproducible.
__device__ int make_frame(const FrameArgs &A, const double p[3], int f[18])
{
    double d0 = __dsub_rn(A.poi[0], p[0]), d1 = __dsub_rn(A.poi[1], p[1]), d2 = __dsub_rn(A.poi[2], p[2]);
    if (d0 == 0.0 && d1 == 0.0 && d2 == 0.0) return NBT_ERR_DEGENERATE;
    if (!(isfinite(d0) && isfinite(d1) && isfinite(d2))) return NBT_ERR_INVALID_ARG;
    double nrm = __dsqrt_rn(dot3_sq(d0, d1, d2));
    double fw[3] = {__ddiv_rn(d0, nrm), __ddiv_rn(d1, nrm), __ddiv_rn(d2, nrm)};
    double c[3] = {fw[1], -fw[0], 0.0};
    double nc = __dsqrt_rn(dot3_sq(c[0], c[1], c[2]));
    if (nc < 1e-6) {
        c[0] = 0.0; c[1] = fw[2]; c[2] = -fw[1];
        nc = __dsqrt_rn(dot3_sq(c[0], c[1], c[2]));
    }
    double rt[3] = {__ddiv_rn(c[0], nc), __ddiv_rn(c[1], nc), __ddiv_rn(c[2], nc)};
    double up[3] = {__dsub_rn(__dmul_rn(rt[1], fw[2]), __dmul_rn(rt[2], fw[1])),
                    __dsub_rn(__dmul_rn(rt[2], fw[0]), __dmul_rn(rt[0], fw[2])),
                    __dsub_rn(__dmul_rn(rt[0], fw[1]), __dmul_rn(rt[1], fw[0]))};
    double s = A.voxel_size;
    double rs = __ddiv_rn(A.range, s);
    double hx = __ddiv_rn(rs, __dmul_rn(2.0, A.cam.fx));
    double hy = __ddiv_rn(rs, __dmul_rn(2.0, A.cam.fy));
    double ch = __dmul_rn(rs, A.cam.tan_half_fov_h);
    double cv = __dmul_rn(rs, A.cam.tan_half_fov_v);
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ok &= rne_q16(__ddiv_rn(__dsub_rn(p[k], A.origin[k]), s), &f[k]);
        ok &= rne_q16(__dmul_rn(rs, fw[k]), &f[3 + k]);
        ok &= rne_q16(__dmul_rn(hx, rt[k]), &f[6 + k]);
        ok &= rne_q16(__dmul_rn(hy, up[k]), &f[9 + k]);
        ok &= rne_q16(__dmul_rn(ch, rt[k]), &f[12 + k]);
        ok &= rne_q16(__dmul_rn(cv, up[k]), &f[15 + k]);
    }
    if (!ok) return NBT_ERR_INVALID_ARG;
    // every ray endpoint must stay inside (-2^30, 2^30): E is affine in the lattice
    // offsets, so checking the four lattice corners (and the corner rays) suffices.
    const long long lim = 1073741824LL;
    long long mw = A.cam.width - 1, mh = A.cam.height - 1;
    for (int q = 0; q < 8; ++q) {
        if (q >= 4 && !A.cam.add_corners) break;
        long long sr = (q & 1) ? 1 : -1, su = (q & 2) ? 1 : -1;
        for (int k = 0; k < 3; ++k) {
            long long e = (long long)f[k] + f[3 + k];
            e += (q < 4) ? sr * mw * f[6 + k] + su * mh * f[9 + k] : sr * f[12 + k] + su * f[15 + k];
            if (e <= -lim || e >= lim) return NBT_ERR_INVALID_ARG;
        }
    }
    return NBT_OK;
}

__global__ void k_persp_frames(FrameArgs A, int32_t *__restrict__ frames, unsigned long long *__restrict__ totals,
                               int *work_counter, int *err)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *work_counter = 0;
    if (i >= A.n) return;
    const double *pp = A.persp + 3 * (size_t)(A.first + (size_t)i * A.stride);
    double p[3] = {pp[0], pp[1], pp[2]};
    int f[18] = {0};
    int st = make_frame(A, p, f);
    int32_t *dst = frames + (size_t)i * kFrameInts;
#pragma unroll
    for (int k = 0; k < 18; ++k) dst[k] = st ? 0 : f[k];
    dst[18] = st;
    dst[19] = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) totals[4 * (size_t)i + k] = 0ull;
    if (st) atomicCAS(err, 0, st);
}

// ------------------------------------------------------------ trace (a5-a8)

struct TraceArgs {
    MapView m;
    const int32_t *__restrict__ frames;
    unsigned long long *totals;
    int *work_counter;
    int W, H, add_corners;
    int tiled;                  // 1: warp-coherent 8x4 pixel tiles
    int Wt;                     // tiles per row
    int n_tile_slots;           // tiles * 32 (tiled) or W*H
    int slots;                  // slots per perspective (incl. 4 corner slots)
    int chunk;                  // slots per chunk (multiple of 32)
    int chunks_per_persp;
    int total_chunks;
};

// Map slot -> lattice offsets (mi, mk) = (2i-(W-1), 2kk-(H-1)) or a corner ray.
__device__ __forceinline__ bool slot_ray(const TraceArgs &T, int slot, int &mi, int &mk, int &corner)
{
    corner = -1;
    int i, kk;
    if (slot >= T.n_tile_slots) {
        corner = slot - T.n_tile_slots;
        return true;
    }
    if (T.tiled) {
        int tile = slot >> 5, l = slot & 31;
        int ty = tile / T.Wt, tx = tile - ty * T.Wt;
        i = tx * 8 + (l & 7);
        kk = ty * 4 + (l >> 3);
        if (i >= T.W || kk >= T.H) return false;
    } else {
        kk = slot / T.W;
        i = slot - kk * T.W;
    }
    mi = 2 * i - (T.W - 1);
    mk = 2 * kk - (T.H - 1);
    return true;
}

__device__ __forceinline__ void ray_endpoint(const int f[18], int mi, int mk, int corner, int e[3])
{
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        uint32_t v;   // modular arithmetic: the true result is inside (-2^30, 2^30)
        if (corner < 0) {
            v = (uint32_t)f[k] + (uint32_t)f[3 + k] + (uint32_t)mi * (uint32_t)f[6 + k] + (uint32_t)mk * (uint32_t)f[9 + k];
        } else {
            uint32_t rc = (uint32_t)f[12 + k], uc = (uint32_t)f[15 + k];
            v = (uint32_t)f[k] + (uint32_t)f[3 + k] + ((corner & 1) ? rc : 0u - rc) + ((corner & 2) ? uc : 0u - uc);
        }
        e[k] = (int)v;
    }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_id_trace(TraceArgs T)
{
    const int lane = threadIdx.x & 31;
    for (;;) {
        int chunk = 0;
        if (lane == 0) chunk = atomicAdd(T.work_counter, 1);
        chunk = __shfl_sync(0xffffffffu, chunk, 0);
        if (chunk >= T.total_chunks) return;
        const int j = chunk / T.chunks_per_persp;
        const int s_begin = (chunk - j * T.chunks_per_persp) * T.chunk;
        const int s_end = min(s_begin + T.chunk, T.slots);
        const int4 *fp = reinterpret_cast<const int4 *>(T.frames + (size_t)j * kFrameInts);
        int4 q0 = __ldg(fp), q1 = __ldg(fp + 1), q2 = __ldg(fp + 2), q3 = __ldg(fp + 3), q4 = __ldg(fp + 4);
        if (q4.z != 0) continue;   // invalid perspective (flagged by k_persp_frames); warp-uniform
        const int f[18] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x,
                           q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w, q4.x, q4.y};
        Counts c{0, 0, 0, 0};
        Ray r;
        bool have = false;
        int slot = s_begin + lane;
        for (;;) {
            if (!have) {
                int mi = 0, mk = 0, corner = -1;
                bool found = false;
                while (slot < s_end) {
                    bool ok = slot_ray(T, slot, mi, mk, corner);
                    slot += 32;
                    if (ok) { found = true; break; }
                }
                if (!found) break;
                int e[3];
                ray_endpoint(f, mi, mk, corner, e);
                ray_setup(r, f, e);
                if (ray_enter<false>(r, T.m, nullptr, nullptr, 0)) {
                    if (T.m.policy == NBT_OUTSIDE_UNKNOWN) c.u += r.pre;
                    continue;
                }
                have = true;
            }
            // one voxel visit + one DDA step of the fast walk
            uint32_t code = code_at(T.m, r.idx);
            if (code >= 2u) {
                uint32_t tail = 0, l;
                if (code == 2u) {
                    l = r.s - r.s0 + 1;
                    c.o += 1;
                    c.u += l - r.nf - 1;
                } else {
                    l = r.s - r.s0;
                    tail = r.n - r.s + 1;
                    c.u += l - r.nf;
                }
                if (T.m.policy == NBT_OUTSIDE_UNKNOWN) c.u += r.pre + tail;
                c.f += r.nf;
                c.l += l;
                have = false;
                continue;
            }
            r.nf += code;
            if (r.s == r.n) {
                uint32_t l = r.s - r.s0 + 1;
                c.u += l - r.nf + (T.m.policy == NBT_OUTSIDE_UNKNOWN ? r.pre : 0);
                c.f += r.nf;
                c.l += l;
                have = false;
                continue;
            }
            int a = ray_advance(r);
            r.idx += (a == 0) ? r.dX : ((a == 1) ? r.dY : r.dZ);
            r.s++;
        }
        // chunk totals: integer, so the summation order cannot change the result
        uint32_t su = __reduce_add_sync(0xffffffffu, c.u);
        uint32_t sf = __reduce_add_sync(0xffffffffu, c.f);
        uint32_t so = __reduce_add_sync(0xffffffffu, c.o);
        uint32_t sl = __reduce_add_sync(0xffffffffu, c.l);
        if (lane == 0) {
            unsigned long long *t = T.totals + 4 * (size_t)j;
            atomicAdd(t + 0, (unsigned long long)su);
            atomicAdd(t + 1, (unsigned long long)sf);
            atomicAdd(t + 2, (unsigned long long)so);
            atomicAdd(t + 3, (unsigned long long)sl);
        }
    }
}

// ------------------------------------------------------------ finalize (a8)

__global__ void k_id_finalize(FrameArgs A, const int32_t *__restrict__ frames,
                              const unsigned long long *__restrict__ totals, double g_u, double g_f, double g_o,
                              double n_e, double *__restrict__ xyz_out, double *__restrict__ gain_out,
                              unsigned long long *__restrict__ counts_out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const double *pp = A.persp + 3 * (size_t)(A.first + (size_t)i * A.stride);
    xyz_out[3 * (size_t)i + 0] = pp[0];
    xyz_out[3 * (size_t)i + 1] = pp[1];
    xyz_out[3 * (size_t)i + 2] = pp[2];
    unsigned long long tu = totals[4 * (size_t)i], tf = totals[4 * (size_t)i + 1];
    unsigned long long to = totals[4 * (size_t)i + 2], tl = totals[4 * (size_t)i + 3];
    double g = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)tu, g_u), __dmul_rn((double)tf, g_f)),
                                   __dmul_rn((double)to, g_o)),
                         n_e);
    if (frames[(size_t)i * kFrameInts + 18] != 0) g = __longlong_as_double(0x7ff8000000000000LL);   // NaN
    gain_out[i] = g;
    if (counts_out) {
        counts_out[4 * (size_t)i + 0] = tu;
        counts_out[4 * (size_t)i + 1] = tf;
        counts_out[4 * (size_t)i + 2] = to;
        counts_out[4 * (size_t)i + 3] = tl;
    }
}

// ------------------------------------------------------------ debug hooks

__global__ void k_debug_trace(MapView m, const int32_t *__restrict__ o, const int32_t *__restrict__ e, int n_rays,
                              int max_visits, int32_t *ijk, uint8_t *code, int32_t *len, uint32_t *counts)
{
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    int oo[3] = {o[3 * r], o[3 * r + 1], o[3 * r + 2]};
    int ee[3] = {e[3 * r], e[3 * r + 1], e[3 * r + 2]};
    Ray ray;
    ray_setup(ray, oo, ee);
    int32_t *ri = ijk + (size_t)r * max_visits * 3;
    uint8_t *rc = code + (size_t)r * max_visits;
    Counts c{0, 0, 0, 0};
    if (ray_enter<true>(ray, m, ri, rc, max_visits)) {
        if (m.policy == NBT_OUTSIDE_UNKNOWN) c.u += ray.pre;
    } else {
        ray_walk<true>(ray, m, c, ri, rc, max_visits);
    }
    // visits recorded: everything up to the stop (or the whole walk)
    len[r] = (c.o ? ray.s + 1 : ray.n + 1);
    counts[4 * r + 0] = c.u; counts[4 * r + 1] = c.f; counts[4 * r + 2] = c.o; counts[4 * r + 3] = c.l;
}

__global__ void k_debug_frames(FrameArgs A, int32_t *out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const double *pp = A.persp + 3 * (size_t)i;
    double p[3] = {pp[0], pp[1], pp[2]};
    int f[18] = {0};
    int st = make_frame(A, p, f);
    for (int k = 0; k < 18; ++k) out[19 * (size_t)i + k] = st ? 0 : f[k];
    out[19 * (size_t)i + 18] = st;
}

MapView view_of(nbt_map m)
{
    MapView v;
    v.words = m->d_words;
    v.nx = m->desc.nx; v.ny = m->desc.ny; v.nz = m->desc.nz;
    v.px = (int)m->px;
    v.pxy = (int)(m->px * m->py);
    v.policy = m->desc.outside_policy;
    return v;
}

FrameArgs frame_args(nbt_map m, const double *d_persp, int32_t first, int32_t stride, int32_t n, const double poi[3],
                     const nbt_camera &cam, double range)
{
    FrameArgs A;
    A.persp = d_persp; A.first = first; A.stride = stride; A.n = n;
    for (int k = 0; k < 3; ++k) { A.poi[k] = poi[k]; A.origin[k] = m->desc.origin[k]; }
    A.voxel_size = m->desc.voxel_size;
    A.range = range;
    A.cam = cam;
    return A;
}

}  // namespace

nbt_status launch_id(nbt_ctx ctx, nbt_map m, const IdLaunch &L)
{
    if (L.n == 0) return NBT_OK;
    nbt_status st;
    if ((st = ctx->frames.ensure((size_t)L.n * kFrameInts * 4))) return st;
    if ((st = ctx->totals.ensure((size_t)L.n * 32))) return st;
    if ((st = ctx->counter.ensure(64))) return st;
    FrameArgs A = frame_args(m, L.d_persp, L.first, L.stride, L.n, L.poi, L.cam, L.range);
    int *counter = ctx->counter.as<int>();
    {
    ProfScope ps(ctx, NBT_KERNEL_FRAMES);
    k_persp_frames<<<(L.n + 127) / 128, 128, 0, ctx->stream>>>(A, ctx->frames.as<int32_t>(),
                                                                ctx->totals.as<unsigned long long>(), counter,
                                                                ctx->d_err);
    NBT_LAUNCHED(ctx);
    }

    TraceArgs T;
    T.m = view_of(m);
    T.frames = ctx->frames.as<int32_t>();
    T.totals = ctx->totals.as<unsigned long long>();
    T.work_counter = counter;
    T.W = L.cam.width; T.H = L.cam.height; T.add_corners = L.cam.add_corners ? 1 : 0;
    T.tiled = (T.W >= 8 && T.H >= 4) ? 1 : 0;
    T.Wt = (T.W + 7) / 8;
    int Ht = (T.H + 3) / 4;
    T.n_tile_slots = T.tiled ? T.Wt * Ht * 32 : T.W * T.H;
    T.slots = T.n_tile_slots + (T.add_corners ? 4 : 0);
    if (ctx->trace_blocks_per_sm == 0) {
        int b = 0;
        NBT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_id_trace, kWarpsPerBlock * 32, 0));
        ctx->trace_blocks_per_sm = b > 0 ? b : 1;
    }
    long long resident_warps = (long long)ctx->num_sms * ctx->trace_blocks_per_sm * kWarpsPerBlock;
    long long total_slots = (long long)L.n * T.slots;
    long long per = total_slots / (8 * resident_warps);          // aim for >= 8 chunks per warp
    int chunk = (int)((per / 32) * 32);
    chunk = chunk < 32 ? 32 : (chunk > 512 ? 512 : chunk);
    T.chunk = chunk;
    T.chunks_per_persp = (T.slots + chunk - 1) / chunk;
    long long tc = (long long)T.chunks_per_persp * L.n;
    if (tc >= (1ll << 31)) return fail(NBT_ERR_INVALID_ARG, "nbt_id_compute: too many rays in one call");
    T.total_chunks = (int)tc;
    long long want_blocks = (tc + kWarpsPerBlock - 1) / kWarpsPerBlock;
    long long max_blocks = (long long)ctx->num_sms * ctx->trace_blocks_per_sm;
    int blocks = (int)(want_blocks < max_blocks ? want_blocks : max_blocks);
    {
        ProfScope ps(ctx, NBT_KERNEL_TRACE);
        k_id_trace<<<blocks, kWarpsPerBlock * 32, 0, ctx->stream>>>(T);
        NBT_LAUNCHED(ctx);
    }

    int ne = L.cam.width * L.cam.height + (L.cam.add_corners ? 4 : 0);
    ProfScope ps(ctx, NBT_KERNEL_FINALIZE);
    k_id_finalize<<<(L.n + 127) / 128, 128, 0, ctx->stream>>>(
        A, ctx->frames.as<int32_t>(), ctx->totals.as<unsigned long long>(), m->desc.gain[0], m->desc.gain[1],
        m->desc.gain[2], (double)ne, L.d_xyz_out, L.d_gain_out,
        reinterpret_cast<unsigned long long *>(L.d_counts_out));
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_debug_trace(nbt_ctx ctx, nbt_map m, const int32_t *d_o, const int32_t *d_e, int32_t n_rays,
                              int32_t max_visits, int32_t *d_ijk, uint8_t *d_code, int32_t *d_len,
                              uint32_t *d_counts)
{
    if (n_rays == 0) return NBT_OK;
    k_debug_trace<<<(n_rays + 127) / 128, 128, 0, ctx->stream>>>(view_of(m), d_o, d_e, n_rays, max_visits, d_ijk,
                                                                 d_code, d_len, d_counts);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_debug_frames(nbt_ctx ctx, nbt_map m, const double poi[3], const double *d_persp, int32_t n,
                               const nbt_camera &cam, double range, int32_t *d_frames)
{
    if (n == 0) return NBT_OK;
    FrameArgs A = frame_args(m, d_persp, 0, 1, n, poi, cam, range);
    k_debug_frames<<<(n + 127) / 128, 128, 0, ctx->stream>>>(A, d_frames);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
