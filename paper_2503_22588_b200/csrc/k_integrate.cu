// Map integration on the device (readings Q33-Q37): the
// step before the ID path, so that a new depth frame updates the voxel map without a
// host round trip (the paper blames host <-> device map traffic for its GPU
// losses at small N_P).
//
//   k_filter_keys     voxel filter, part 1 (Q33): one 63-bit cell key per point,
//                     (iz, iy, ix) from high to low bits so that key order is the output
//                     order; non-finite or out-of-range points poison the cloud.
//   (cub)             stable radix sort of (key, input index), run-length encoding of
//                     the keys, exclusive scan of the run lengths.
//   k_filter_centroid one thread per cell: the centroid, summed in input order (the sort
//                     is stable) -- bit-identical to a sequential loop.
//   k_integrate_rays  one thread per sensor ray: range cut, both ends to Q12
//                     (Q34), the exact DDA of the ID walk (dda.cuh, Q13) over every
//                     visited voxel; each in-grid voxel gets its flag byte OR-ed with
//                     1 (visited) or 3 (ray ends here with a hit).  The first flag of a
//                     voxel appends it to the touched list (warp-aggregated atomics), so
//                     the update pass visits each voxel exactly once (Q35).
//   k_integrate_apply one thread per touched voxel: the log-odds update in float (Q36),
//                     the state and probability level (Q37), the write into the ID's
//                     packed map store (same field-xor as the a2 delta path), the a2
//                     delta when (state, level) changed, and the flag reset.
//
// Flags live in a dense x-fastest byte array that the apply pass leaves zeroed, so no
// per-cloud clear of the whole grid is needed.  A poisoned cloud (invalid point, Q12
// overflow) updates nothing: the apply pass only clears the flags it finds.
#include <math.h>

#include <cub/cub.cuh>

#include "dda.cuh"
#include "map_store.cuh"
#include "nbt_internal.cuh"

namespace nbt {
namespace {

using dda::Walk;

constexpr double kKeyLimit = 1048576.0;          // |cell index| < 2^20 (Q33)
constexpr uint64_t kBadKey = ~0ull;
constexpr double kQ12Limit = 1073741824.0;       // |Q12 coordinate| < 2^30 (Q19)
constexpr int kWideRayVoxels = 700;              // int32 DDA terms up to this many voxels per axis

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Append v to list[] with one atomic per converged group of lanes.
__device__ __forceinline__ void append(uint32_t *list, uint32_t *count, uint32_t v)
{
    const unsigned m = __activemask();
    const int leader = __ffs(m) - 1;
    const unsigned rank = __popc(m & ((1u << lane_id()) - 1u));
    uint32_t base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(count, (uint32_t)__popc(m));
    base = __shfl_sync(m, base, leader);
    list[base + rank] = v;
}

// ------------------------------------------------------------------ voxel filter

__global__ void k_filter_keys(const double *__restrict__ pts, uint32_t n, double leaf,
                              unsigned long long *__restrict__ keys, uint32_t *__restrict__ idx, int *bad,
                              int *err)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned long long key = 0;
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double v = pts[3 * (size_t)i + a];
            const double c = floor(__ddiv_rn(v, leaf));
            ok = ok && isfinite(v) && fabs(c) < kKeyLimit;
            if (ok) key |= (unsigned long long)((long long)c + (1ll << 20)) << (21 * a);
        }
        if (!ok) {
            key = kBadKey;
            atomicExch(bad, 1);
            atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
        }
        keys[i] = key;
        idx[i] = i;
    }
}

// Cells c < *n_runs (the last run is the poison key if any point was invalid).
__global__ void k_filter_centroid(const double *__restrict__ pts, const uint32_t *__restrict__ idx_sorted,
                                  const unsigned long long *__restrict__ run_keys,
                                  const uint32_t *__restrict__ run_len, const uint32_t *__restrict__ run_off,
                                  const uint32_t *__restrict__ n_runs, double *__restrict__ out,
                                  int32_t *__restrict__ out_count, uint32_t *__restrict__ n_out)
{
    const uint32_t runs = *n_runs;
    const uint32_t m = (runs > 0 && run_keys[runs - 1] == kBadKey) ? runs - 1 : runs;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = m;
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x) {
        const uint32_t b = run_off[c], len = run_len[c];
        double sx = 0.0, sy = 0.0, sz = 0.0;
        for (uint32_t k = 0; k < len; ++k) {
            const size_t p = 3 * (size_t)idx_sorted[b + k];
            sx = __dadd_rn(sx, pts[p]);
            sy = __dadd_rn(sy, pts[p + 1]);
            sz = __dadd_rn(sz, pts[p + 2]);
        }
        const double dn = (double)len;
        out[3 * (size_t)c] = __ddiv_rn(sx, dn);
        out[3 * (size_t)c + 1] = __ddiv_rn(sy, dn);
        out[3 * (size_t)c + 2] = __ddiv_rn(sz, dn);
        if (out_count) out_count[c] = (int32_t)len;
    }
}

// ------------------------------------------------------------------ integration

struct RayArgs {
    double sensor[3];
    double org[3];          // map origin (world)
    double s;               // voxel size
    double max_range;       // <= 0: unlimited
    int nx, ny, nz;
};

__device__ __forceinline__ bool to_q12(double x, double org, double s, int &out)
{
    const double q = __dmul_rn(__ddiv_rn(__dsub_rn(x, org), s), 4096.0);
    if (!(fabs(q) < kQ12Limit)) return false;
    out = (int)rint(q);
    return true;
}

__device__ __forceinline__ void mark(uint32_t *flags, uint32_t *touched, uint32_t *n_touched, uint32_t v,
                                     uint32_t want)
{
    uint32_t *w = flags + (v >> 2);
    const uint32_t sh = (v & 3u) * 8u;
    if (((__ldcg(w) >> sh) & want) == want) return;     // already marked (a stale read only costs an atomic)
    const uint32_t old = atomicOr(w, want << sh);
    if (((old >> sh) & 0xffu) == 0u) append(touched, n_touched, v);
}

template <typename T>
__global__ void __launch_bounds__(256) k_integrate_rays(const double *__restrict__ rays, const uint32_t *n_rays_dev,
                                                        uint32_t n_rays_host, RayArgs a, uint32_t *flags,
                                                        uint32_t *touched, uint32_t *n_touched, int *bad, int *err)
{
    const uint32_t n = n_rays_dev ? *n_rays_dev : n_rays_host;
    if (*bad) return;
    int o12[3];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) ok = ok && to_q12(a.sensor[k], a.org[k], a.s, o12[k]);
    dda::MapView mv{};
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double p[3] = {rays[3 * (size_t)i], rays[3 * (size_t)i + 1], rays[3 * (size_t)i + 2]};
        double d[3], q[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) { d[k] = __dsub_rn(p[k], a.sensor[k]); q[k] = p[k]; }
        const double dist =
            __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
        uint32_t hit = 3u;
        if (a.max_range > 0.0 && dist > a.max_range) {          // cut at the range, carve only
            const double f = __ddiv_rn(a.max_range, dist);
#pragma unroll
            for (int k = 0; k < 3; ++k) q[k] = __dadd_rn(a.sensor[k], __dmul_rn(d[k], f));
            hit = 1u;
        }
        int e12[3];
        bool rok = ok;
#pragma unroll
        for (int k = 0; k < 3; ++k) rok = rok && to_q12(q[k], a.org[k], a.s, e12[k]);
        if (!rok) {
            atomicExch(bad, 1);
            atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
            continue;
        }
        Walk<T> w;
        dda::walk_setup(w, o12, e12);
        w.dX = w.dY = w.ndZ = 0;
        w.idx = 0;
        for (int s = 0;; ++s) {
            if ((unsigned)w.vx < (unsigned)a.nx && (unsigned)w.vy < (unsigned)a.ny && (unsigned)w.vz < (unsigned)a.nz) {
                const uint32_t v = (uint32_t)w.vx + (uint32_t)a.nx * ((uint32_t)w.vy + (uint32_t)a.ny * (uint32_t)w.vz);
                mark(flags, touched, n_touched, v, s == w.n ? hit : 1u);
            }
            if (s == w.n) break;
            dda::walk_step<T, kLayoutLinear, true>(w, mv);
        }
    }
}

struct ApplyArgs {
    float lh, lm, lo, hi;        // L_hit, L_miss, clamp (Q36)
    float th_occ, th_free;       // logit(t_occ), logit(t_free) (Q37)
    float phi[64];               // level boundaries logit((k - 1/2)/63), k = 1..63
    int nx, ny;
};

__device__ __forceinline__ void classify(float l, const ApplyArgs &a, uint32_t &code, uint32_t &level)
{
    code = (l >= a.th_occ) ? 2u : (l <= a.th_free ? 1u : 0u);
    uint32_t lv = 0;
#pragma unroll 7
    for (int k = 0; k < 63; ++k) lv += (l >= a.phi[k]) ? 1u : 0u;
    level = lv;
}

__global__ void __launch_bounds__(256) k_integrate_apply(const uint32_t *__restrict__ touched,
                                                         const uint32_t *n_touched, uint8_t *flags8, float *L,
                                                         ApplyArgs a, Geom g, uint32_t *words, uint32_t *d_idx,
                                                         uint16_t *d_val, uint32_t *n_deltas, const int *bad)
{
    const uint32_t n = *n_touched;
    const bool poisoned = *bad != 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t v = touched[t];
        const uint32_t f = flags8[v];
        flags8[v] = 0;
        if (poisoned) continue;
        const float l0 = L[v];
        const bool observed = !isnan(l0);
        float l1 = __fadd_rn(observed ? l0 : 0.0f, (f & 2u) ? a.lh : a.lm);
        l1 = fminf(fmaxf(l1, a.lo), a.hi);
        L[v] = l1;
        uint32_t c0 = 0, lv0 = 0, c1, lv1;
        if (observed) classify(l0, a, c0, lv0);
        classify(l1, a, c1, lv1);
        if (c0 == c1 && lv0 == lv1) continue;
        const uint32_t x = v % (uint32_t)a.nx, r = v / (uint32_t)a.nx;
        const uint32_t y = r % (uint32_t)a.ny, z = r / (uint32_t)a.ny;
        if (words) {
            const uint64_t pi = store_index(g, x, y, z);
            uint32_t *w = words + word_of(g, pi);
            const uint32_t sh = shift_of(g, pi);
            const uint32_t mask = g.vbits == 2 ? 3u : 0xffu;
            const uint32_t nw = stored_value(g, c1, lv1);
            const uint32_t old = (*(volatile uint32_t *)w >> sh) & mask;
            if (old != nw) atomicXor(w, (old ^ nw) << sh);
        }
        const unsigned m = __activemask();
        const int leader = __ffs(m) - 1;
        const unsigned rank = __popc(m & ((1u << lane_id()) - 1u));
        uint32_t base = 0;
        if ((int)lane_id() == leader) base = atomicAdd(n_deltas, (uint32_t)__popc(m));
        base = __shfl_sync(m, base, leader);
        d_idx[base + rank] = v;
        d_val[base + rank] = (uint16_t)(c1 | (lv1 << 8));
    }
}

inline unsigned grid_for(nbt_ctx ctx, size_t n, unsigned threads, unsigned per_sm)
{
    const size_t want = (n + threads - 1) / threads;
    const size_t cap = (size_t)ctx->num_sms * per_sm;
    return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

float logit_f(double p) { return (float)log(p / (1.0 - p)); }

}  // namespace

nbt_status launch_voxel_filter(nbt_ctx ctx, nbt_occ_s *o, const double *d_pts, uint32_t n, double leaf,
                               int32_t *d_count_out)
{
    nbt_status st;
    if ((st = o->keys.ensure((size_t)n * 8)) || (st = o->keys_alt.ensure((size_t)n * 8)) ||
        (st = o->idx.ensure((size_t)n * 4)) || (st = o->idx_alt.ensure((size_t)n * 4)) ||
        (st = o->runs.ensure((size_t)n * 8 + 16)) || (st = o->filtered.ensure((size_t)n * 24)))
        return st;
    auto *keys = o->keys.as<unsigned long long>(), *keys_s = o->keys_alt.as<unsigned long long>();
    auto *idx = o->idx.as<uint32_t>(), *idx_s = o->idx_alt.as<uint32_t>();
    uint32_t *run_len = o->runs.as<uint32_t>(), *run_off = run_len + n, *n_runs = run_off + n;
    k_filter_keys<<<grid_for(ctx, n, 256, 8), 256, 0, ctx->stream>>>(d_pts, n, leaf, keys, idx, o->d_ctl + kOccBad,
                                                                      ctx->d_err);
    NBT_LAUNCHED(ctx);
    size_t t1 = 0, t2 = 0, t3 = 0;
    NBT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys_s, idx, idx_s, (int)n, 0, 64, ctx->stream));
    NBT_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t2, keys_s, keys, run_len, n_runs, (int)n, ctx->stream));
    NBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t3, run_len, run_off, (int)n, ctx->stream));
    size_t tmp = t1 > t2 ? t1 : t2;
    tmp = tmp > t3 ? tmp : t3;
    if ((st = o->cub_tmp.ensure(tmp))) return st;
    NBT_CUDA(cub::DeviceRadixSort::SortPairs(o->cub_tmp.p, tmp, keys, keys_s, idx, idx_s, (int)n, 0, 64,
                                             ctx->stream));
    // run keys overwrite the unsorted keys (no longer needed)
    NBT_CUDA(cub::DeviceRunLengthEncode::Encode(o->cub_tmp.p, tmp, keys_s, keys, run_len, n_runs, (int)n,
                                                ctx->stream));
    NBT_CUDA(cub::DeviceScan::ExclusiveSum(o->cub_tmp.p, tmp, run_len, run_off, (int)n, ctx->stream));
    k_filter_centroid<<<grid_for(ctx, n, 256, 8), 256, 0, ctx->stream>>>(
        d_pts, idx_s, keys, run_len, run_off, n_runs, o->filtered.as<double>(), d_count_out,
        reinterpret_cast<uint32_t *>(o->d_ctl + kOccRays));
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_integrate(nbt_ctx ctx, nbt_occ_s *o, nbt_map m, const double sensor[3], const double *d_pts,
                            uint32_t n, const nbt_integrate_params &p)
{
    nbt_status st;
    ProfScope ps(ctx, NBT_KERNEL_INTEGRATE);
    // per-call control words: bad flag, ray count, touched count, delta count
    NBT_CUDA(cudaMemsetAsync(o->d_ctl, 0, kOccCtlInts * sizeof(int), ctx->stream));
    const double *rays = d_pts;
    const uint32_t *n_rays_dev = nullptr;      // filtered: the cell count is known on the device only
    o->last_points = n;
    o->last_filtered = p.leaf > 0.0;
    if (p.leaf > 0.0 && n > 0) {
        if ((st = launch_voxel_filter(ctx, o, d_pts, n, p.leaf, nullptr))) return st;
        rays = o->filtered.as<double>();
        n_rays_dev = reinterpret_cast<const uint32_t *>(o->d_ctl + kOccRays);
    }
    RayArgs ra;
    for (int k = 0; k < 3; ++k) { ra.sensor[k] = sensor[k]; ra.org[k] = o->desc.origin[k]; }
    ra.s = o->desc.voxel_size;
    ra.max_range = p.max_range;
    ra.nx = o->desc.nx; ra.ny = o->desc.ny; ra.nz = o->desc.nz;
    const bool wide = !(p.max_range > 0.0 && p.max_range / o->desc.voxel_size + 2.0 < (double)kWideRayVoxels);
    uint32_t *ctl = reinterpret_cast<uint32_t *>(o->d_ctl);
    const unsigned gr = grid_for(ctx, n, 256, 8);
    if (n > 0) {
        if (wide)
            k_integrate_rays<long long><<<gr, 256, 0, ctx->stream>>>(rays, n_rays_dev, n, ra, o->d_flags,
                                                                     o->d_touched, ctl + kOccTouched,
                                                                     o->d_ctl + kOccBad, ctx->d_err);
        else
            k_integrate_rays<int><<<gr, 256, 0, ctx->stream>>>(rays, n_rays_dev, n, ra, o->d_flags, o->d_touched,
                                                               ctl + kOccTouched, o->d_ctl + kOccBad, ctx->d_err);
        NBT_LAUNCHED(ctx);
    }
    ApplyArgs aa;
    aa.lh = logit_f(p.p_hit); aa.lm = logit_f(p.p_miss);
    aa.lo = logit_f(p.p_min); aa.hi = logit_f(p.p_max);
    aa.th_occ = logit_f(p.t_occ); aa.th_free = logit_f(p.t_free);
    for (int k = 1; k <= 63; ++k) aa.phi[k - 1] = logit_f((k - 0.5) / 63.0);
    aa.phi[63] = INFINITY;
    aa.nx = o->desc.nx; aa.ny = o->desc.ny;
    Geom g{};
    uint32_t *words = nullptr;
    if (m) { g = geom_of(m); words = m->d_words; }
    k_integrate_apply<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(
        o->d_touched, ctl + kOccTouched, reinterpret_cast<uint8_t *>(o->d_flags), o->d_L, aa, g, words, o->d_didx,
        o->d_dval, ctl + kOccDeltas, o->d_ctl + kOccBad);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
