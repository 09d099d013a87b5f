// Map integration on the device (readings Q33-Q37): the
// step before the ID path, so that a new depth frame updates the voxel map without a
// host round trip (the paper blames host <-> device map traffic for its GPU
// losses at small N_P).
//
//   k_filter_keys     voxel filter, part 1 (Q33): one 48-bit cell key per point,
//                     (iz, iy, ix) from high to low bits so that key order is the output
//                     order; non-finite or out-of-range points poison the cloud.
//   (cub)             stable radix sort of (key, input index).
//   k_filter_gather   the points in cell order, cell heads flagged; (cub) select of the
//                     head positions = the cell offsets.
//   k_filter_centroid 8 lanes per cell: the centroid of its contiguous run, summed in input
//                     order (the sort is stable) -- bit-identical to a sequential loop.
//   k_integrate_rays  one thread per piece of a sensor ray (exact split, see below): range
//                     cut, both ends to Q16
//                     (Q34), the exact DDA of the ID walk (dda.cuh, Q13) over every
//                     visited voxel, whose flag byte gets 1 (visited) or 3 (the ray ends
//                     here with a hit) OR-ed in with fire-and-forget atomics (Q35: each
//                     voxel's update depends only on the OR of its flags, not on ray order).
//   k_integrate_collect dense scan of the flag bytes, 16 per load: lists every flagged voxel
//                     (with its hit bit) and clears the flags.
//   k_integrate_apply one thread per listed voxel: the log-odds update in float (Q36), the
//                     state and probability level (Q37), the write into the ID's packed map
//                     store, the a2 delta when (state, level) changed.
//
// The apply pass leaves the flags zeroed, so no per-cloud clear is needed.  A poisoned
// cloud (invalid point, Q16 overflow) updates nothing: the apply pass only clears flags.
#include <math.h>
#include <stdlib.h>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "dda.cuh"
#include "map_store.cuh"
#include "nbt_internal.cuh"

namespace nbt {
namespace {

using dda::Walk;

constexpr double kKeyLimit = 32767.0;            // |cell index| < 2^15 - 1 (Q33)
constexpr int kKeyBits = 48;                     // 16 bits per axis: 6 radix passes instead of 8
constexpr uint64_t kBadKey = (1ull << kKeyBits) - 1;   // above every valid key (fields <= 0xFFFE)
constexpr double kQ16Limit = 1073741824.0;       // |Q16 coordinate| < 2^30 (Q19)
constexpr int kWideRayVoxels = 16000;            // int32 DDA terms below this many voxels per axis (k_id.cu: < 16383)

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

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
            if (ok) key |= (unsigned long long)((long long)c + (1ll << 15)) << (16 * a);
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

// After the stable sort: the points in cell order (coalesced later reads), the first point
// of every valid cell flagged, and the number of valid points (poisoned keys sort last).
__global__ void k_filter_gather(const double *__restrict__ pts, const uint32_t *__restrict__ idx_sorted,
                                const unsigned long long *__restrict__ keys_sorted, uint32_t n,
                                double *__restrict__ sorted, uint8_t *__restrict__ head, uint32_t *n_valid)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = keys_sorted[i];
        const bool valid = k != kBadKey;
        if (valid) {
            const size_t p = 3 * (size_t)idx_sorted[i];
            sorted[3 * (size_t)i] = pts[p];
            sorted[3 * (size_t)i + 1] = pts[p + 1];
            sorted[3 * (size_t)i + 2] = pts[p + 2];
        }
        head[i] = valid && (i == 0 || keys_sorted[i - 1] != k);
        if (valid && (i + 1 == n || keys_sorted[i + 1] == kBadKey)) *n_valid = i + 1;
    }
}

// One group of 8 lanes per cell: the lanes load the cell's contiguous points 8 at a time
// (independent loads), and every lane of the group adds them in order through shuffles, so
// the sum is the sequential loop's in input order (the sort is stable), bit for bit.
constexpr int kCentroidLanes = 8;

__global__ void __launch_bounds__(256) k_filter_centroid(const double *__restrict__ sorted,
                                                         const uint32_t *__restrict__ run_off,
                                                         const uint32_t *__restrict__ n_runs,
                                                         const uint32_t *__restrict__ n_valid,
                                                         double *__restrict__ out, int32_t *__restrict__ out_count,
                                                         uint32_t *__restrict__ n_out)
{
    const uint32_t m = *n_runs, nv = *n_valid;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = m;
    const uint32_t sub = threadIdx.x & (kCentroidLanes - 1);
    const uint32_t groups = gridDim.x * (blockDim.x / kCentroidLanes);
    // every lane of a warp runs the same number of outer iterations (shuffles need them all)
    const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / kCentroidLanes;
    const uint32_t warp_g0 = g0 - (lane_id() / kCentroidLanes);
    for (uint32_t cw = warp_g0; cw < m; cw += groups) {
        const uint32_t c = cw + lane_id() / kCentroidLanes;
        const bool live = c < m;
        const uint32_t b = live ? run_off[c] : 0u;
        const uint32_t e = live ? (c + 1 < m ? run_off[c + 1] : nv) : 0u;
        const uint32_t len = e - b;
        uint32_t rounds = (len + kCentroidLanes - 1) / kCentroidLanes;
        rounds = __reduce_max_sync(0xffffffffu, rounds);
        double sx = 0.0, sy = 0.0, sz = 0.0;
        for (uint32_t r = 0; r < rounds; ++r) {
            const uint32_t k = b + r * kCentroidLanes + sub;
            double x = 0.0, y = 0.0, z = 0.0;
            if (k < e) {
                x = sorted[3 * (size_t)k];
                y = sorted[3 * (size_t)k + 1];
                z = sorted[3 * (size_t)k + 2];
            }
#pragma unroll
            for (int j = 0; j < kCentroidLanes; ++j) {
                const double xj = __shfl_sync(0xffffffffu, x, j, kCentroidLanes);
                const double yj = __shfl_sync(0xffffffffu, y, j, kCentroidLanes);
                const double zj = __shfl_sync(0xffffffffu, z, j, kCentroidLanes);
                if (r * kCentroidLanes + j < len) {
                    sx = __dadd_rn(sx, xj);
                    sy = __dadd_rn(sy, yj);
                    sz = __dadd_rn(sz, zj);
                }
            }
        }
        if (live && sub == 0) {
            const double dn = (double)len;
            out[3 * (size_t)c] = __ddiv_rn(sx, dn);
            out[3 * (size_t)c + 1] = __ddiv_rn(sy, dn);
            out[3 * (size_t)c + 2] = __ddiv_rn(sz, dn);
            if (out_count) out_count[c] = (int32_t)len;
        }
    }
}

// ------------------------------------------------------- voxel filter by hashing (integration)
// The integration only needs each cell's centroid, not the cells in key order (the rays are
// applied as a set, Q35), so it groups points with a hash table instead of a full sort:
// insert each point's cell key (linear probing, atomicCAS), count per slot and keep its
// lowest point index, scan the counts, scatter point indices into their slot's segment
// (arbitrary order), then place each point at its rank among the segment's indices -- the
// segment holds its points in input order, so the centroid is the same in-order sum as the
// sort path's, bit for bit.  Ranking by scanning the segment costs O(len) per point, so cells
// of more than kBigCell points skip it and their centroid group sums them by walking the input
// in order from the cell's first point: a frame whose points share few cells stays far from
// quadratic (a stable radix sort by slot instead of the ranking was robust too but made every
// camera frame 30% slower).

constexpr unsigned long long kEmptyKey = ~0ull;

// Multiplicative (Fibonacci) hash: the live cells spread over the whole table, so the
// insertion atomics spread over the L2 slices.
__device__ __forceinline__ uint32_t hash_slot(unsigned long long key, int log2cap)
{
    return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - log2cap));
}

constexpr uint32_t kBigCell = 512;    // cells with more points: ordered warp walk, no ranking

__global__ void k_hash_insert(const double *__restrict__ pts, uint32_t n, double leaf, int log2cap,
                              unsigned long long *table, uint32_t *count, uint32_t *first_inv,
                              uint32_t *__restrict__ slot_of, int *bad, int *err)
{
    const uint32_t mask = (1u << log2cap) - 1u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned long long key = 0;
        bool ok = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double v = pts[3 * (size_t)i + a];
            const double c = floor(__ddiv_rn(v, leaf));
            ok = ok && isfinite(v) && fabs(c) < kKeyLimit;
            if (ok) key |= (unsigned long long)((long long)c + (1ll << 15)) << (16 * a);
        }
        if (!ok) {
            slot_of[i] = 0xffffffffu;
            atomicExch(bad, 1);
            atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
            continue;
        }
        // neighbouring pixels share cells: one insertion and one count update per distinct
        // key among the converged lanes
        const unsigned am = __activemask();
        const unsigned peers = __match_any_sync(am, key);
        const int leader = __ffs(peers) - 1;
        uint32_t h = 0;
        if ((int)lane_id() == leader) {
            h = hash_slot(key, log2cap);
            for (;;) {
                const unsigned long long prev = atomicCAS(table + h, kEmptyKey, key);
                if (prev == kEmptyKey || prev == key) break;
                h = (h + 1u) & mask;
            }
            atomicAdd(count + h, (uint32_t)__popc(peers));
            atomicMax(first_inv + h, ~i);            // ~(lowest index); the leader holds the peers' lowest
        }
        h = __shfl_sync(peers, h, leader);
        slot_of[i] = h;
    }
}

__global__ void k_hash_scatter(const uint32_t *__restrict__ slot_of, uint32_t n, const uint32_t *__restrict__ off,
                               const uint32_t *__restrict__ count, uint32_t *fill, uint32_t *__restrict__ seg)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t h = slot_of[i];
        if (h == 0xffffffffu || count[h] > kBigCell) continue;
        seg[off[h] + atomicAdd(fill + h, 1u)] = i;
    }
}

// Also flags the first (lowest-index) point of every cell: selecting the slots of those
// points in index order lists the cells in the order of the depth image's pixels, so the
// rays reach the ray kernel spatially coherent (its flag atomics depend on that) and in a
// deterministic order.
__global__ void k_hash_place(const double *__restrict__ pts, const uint32_t *__restrict__ slot_of, uint32_t n,
                             const uint32_t *__restrict__ off, const uint32_t *__restrict__ count,
                             const uint32_t *__restrict__ first_inv, const uint32_t *__restrict__ seg,
                             double *__restrict__ sorted, uint8_t *__restrict__ head)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t h = slot_of[i];
        head[i] = 0;
        if (h == 0xffffffffu) continue;
        head[i] = first_inv[h] == ~i;
        const uint32_t b = off[h], len = count[h];
        if (len > kBigCell) continue;                 // summed by an ordered walk (k_hash_centroid)
        uint32_t rank = 0;
        for (uint32_t k = 0; k < len; ++k) rank += seg[b + k] < i ? 1u : 0u;
        const size_t d = 3 * (size_t)(b + rank);
        sorted[d] = pts[3 * (size_t)i];
        sorted[d + 1] = pts[3 * (size_t)i + 1];
        sorted[d + 2] = pts[3 * (size_t)i + 2];
    }
}

// Cell c = occupied slot cells[c]: run [off, off + count) of the placed points; the same
// 8-lane in-order sum as k_filter_centroid.  A cell of more than kBigCell points (not placed)
// is summed by its 8-lane group walking the INPUT in order from the cell's first point, 8
// points per step: the group's points of a step (ballot) are added in lane order through
// shuffles -- the same sequential in-order sum -- until all the cell's points are in.
__global__ void __launch_bounds__(256) k_hash_centroid(const double *__restrict__ sorted,
                                                       const double *__restrict__ pts,
                                                       const uint32_t *__restrict__ slot_of, uint32_t n,
                                                       const uint32_t *__restrict__ cells,
                                                       const uint32_t *__restrict__ n_cells,
                                                       const uint32_t *__restrict__ off,
                                                       const uint32_t *__restrict__ count,
                                                       const uint32_t *__restrict__ first_inv,
                                                       double *__restrict__ out, uint32_t *__restrict__ n_out)
{
    const unsigned full = 0xffffffffu;
    const uint32_t m = *n_cells;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = m;
    const uint32_t sub = threadIdx.x & (kCentroidLanes - 1);
    const uint32_t group_shift = lane_id() & ~(kCentroidLanes - 1);
    const uint32_t groups = gridDim.x * (blockDim.x / kCentroidLanes);
    const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / kCentroidLanes;
    const uint32_t warp_g0 = g0 - (lane_id() / kCentroidLanes);
    for (uint32_t cw = warp_g0; cw < m; cw += groups) {
        const uint32_t c = cw + lane_id() / kCentroidLanes;
        const bool live = c < m;
        const uint32_t h = live ? cells[c] : 0u;
        const uint32_t len_all = live ? count[h] : 0u;
        const bool bigc = len_all > kBigCell;
        const uint32_t b = live && !bigc ? off[h] : 0u;
        const uint32_t len = bigc ? 0u : len_all;
        const uint32_t e = b + len;
        uint32_t rounds = (len + kCentroidLanes - 1) / kCentroidLanes;
        rounds = __reduce_max_sync(full, rounds);
        double sx = 0.0, sy = 0.0, sz = 0.0;
        for (uint32_t r = 0; r < rounds; ++r) {
            const uint32_t k = b + r * kCentroidLanes + sub;
            double x = 0.0, y = 0.0, z = 0.0;
            if (k < e) {
                x = sorted[3 * (size_t)k];
                y = sorted[3 * (size_t)k + 1];
                z = sorted[3 * (size_t)k + 2];
            }
#pragma unroll
            for (int j = 0; j < kCentroidLanes; ++j) {
                const double xj = __shfl_sync(full, x, j, kCentroidLanes);
                const double yj = __shfl_sync(full, y, j, kCentroidLanes);
                const double zj = __shfl_sync(full, z, j, kCentroidLanes);
                if (r * kCentroidLanes + j < len) {
                    sx = __dadd_rn(sx, xj);
                    sy = __dadd_rn(sy, yj);
                    sz = __dadd_rn(sz, zj);
                }
            }
        }
        if (__any_sync(full, bigc)) {                  // rare: ordered walk over the input
            uint32_t base = bigc ? ~first_inv[h] : n, done = 0;
            while (__any_sync(full, bigc && done < len_all && base < n)) {
                const bool act = bigc && done < len_all && base < n;
                const uint32_t i = base + sub;
                const bool mine = act && i < n && slot_of[i] == h;
                double x = 0.0, y = 0.0, z = 0.0;
                if (mine) {
                    x = pts[3 * (size_t)i];
                    y = pts[3 * (size_t)i + 1];
                    z = pts[3 * (size_t)i + 2];
                }
                const uint32_t bits = (__ballot_sync(full, mine) >> group_shift) & 0xffu;
                done += __popc(bits);
#pragma unroll
                for (int j = 0; j < kCentroidLanes; ++j) {
                    const double xj = __shfl_sync(full, x, j, kCentroidLanes);
                    const double yj = __shfl_sync(full, y, j, kCentroidLanes);
                    const double zj = __shfl_sync(full, z, j, kCentroidLanes);
                    if ((bits >> j) & 1u) {
                        sx = __dadd_rn(sx, xj);
                        sy = __dadd_rn(sy, yj);
                        sz = __dadd_rn(sz, zj);
                    }
                }
                base += kCentroidLanes;
            }
        }
        if (live && sub == 0) {
            const double dn = (double)len_all;
            out[3 * (size_t)c] = __ddiv_rn(sx, dn);
            out[3 * (size_t)c + 1] = __ddiv_rn(sy, dn);
            out[3 * (size_t)c + 2] = __ddiv_rn(sz, dn);
        }
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

__device__ __forceinline__ bool to_q16(double x, double org, double s, int &out)
{
    const double q = __dmul_rn(__ddiv_rn(__dsub_rn(x, org), s), 65536.0);
    if (!(fabs(q) < kQ16Limit)) return false;
    out = (int)rint(q);
    return true;
}

// Marking: a ray ORs 1 (visited) or 3 (ends here with a hit) into each in-grid voxel's
// flag byte with fire-and-forget atomics -- nothing in the walk waits on memory.  A thread
// skips the OR when its previous one already set those bits in the same word (steps along
// x stay in one 4-voxel word).  All rays start at the sensor and advance in lockstep, so
// the voxels near it would take one atomic per ray: there the lanes of a warp that hit the
// same word combine their bits first (one atomic per word per warp).
//
// Exact ray split.  A frame has only ~30 k rays of ~100-200 steps: one thread per ray
// leaves the GPU latency-bound.  The walk's decision terms are linear in the per-axis
// event counts (c_x, c_y, c_z) -- q_ab = q_ab(0) + c_a |D_b| - c_b |D_a| (dda.cuh) -- and
// q_ab(c_a, c_b) < 0 says exactly that a-event #(c_a + 1) precedes b-event #(c_b + 1).  So
// the state right after the k-th event of the dominant axis A is known in closed form:
// c_A = k, and for every other axis b, c_b = the number of b-events ordered before A's
// k-th (a floor / ceil division of the same terms, clamped to b's event total).  A ray is
// cut into pieces of kPieceEvents A-events; one thread walks one piece from its exact
// start state to the next piece's start.
constexpr int kDedupSteps = 32;
constexpr int kRayThreads = 256;
#ifndef NBT_PIECE_EVENTS
#define NBT_PIECE_EVENTS 24
#endif
#ifndef NBT_PIECE_SLOTS
#define NBT_PIECE_SLOTS 8
#endif
constexpr int kPieceEvents = NBT_PIECE_EVENTS;            // dominant-axis events per piece
constexpr int kPieceSlots = NBT_PIECE_SLOTS;              // threads per ray (pieces j, j + 8, ...)

__device__ __forceinline__ long long floor_div_ll(long long a, long long b)   // b > 0
{
    const long long q = a / b;
    return (q * b > a) ? q - 1 : q;
}

__device__ __forceinline__ long long clamp_ll(long long v, long long hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

// Event counts (c_x, c_y, c_z) right after the k-th event of axis A (k >= 1).
template <typename T>
__device__ __forceinline__ void counts_after(const Walk<T> &w0, int A, long long k, const long long ne[3],
                                             long long c[3])
{
    const long long ad[3] = {(long long)w0.ax, (long long)w0.ay, (long long)w0.az};
    const long long q[3][3] = {{0, (long long)w0.qxy, (long long)w0.qxz},
                               {0, 0, (long long)w0.qyz},
                               {0, 0, 0}};
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        if (b == A) { c[b] = k; continue; }
        if (ad[b] == 0) { c[b] = 0; continue; }
        if (b > A) {      // pair (A, b): b-event #j precedes A-event #k iff q_Ab(k-1, j-1) >= 0
            c[b] = clamp_ll(floor_div_ll(q[A][b] + (k - 1) * ad[b], ad[A]) + 1, ne[b]);
        } else {          // pair (b, A): b-event #j precedes A-event #k iff q_bA(j-1, k-1) < 0,
                          // i.e. (j-1) |D_A| < (k-1) |D_b| - q_bA(0): ceil division
            c[b] = clamp_ll(-floor_div_ll(q[b][A] - (k - 1) * ad[b], ad[A]), ne[b]);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kRayThreads) k_integrate_rays(const double *__restrict__ rays,
                                                                const uint32_t *n_rays_dev, uint32_t n_rays_host,
                                                                RayArgs a, uint32_t *flags, int *bad, int *err)
{
    const uint32_t n = n_rays_dev ? *n_rays_dev : n_rays_host;
    const uint64_t work = (uint64_t)n * kPieceSlots;      // thread t: slot t / n, ray t % n
    if (*bad || (uint64_t)blockIdx.x * blockDim.x >= work) return;
    int o16[3];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) ok = ok && to_q16(a.sensor[k], a.org[k], a.s, o16[k]);
    dda::MapView mv{};
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < work; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t slot = (uint32_t)(t / n), i = (uint32_t)(t % n);
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
        int e16[3];
        bool rok = ok;
#pragma unroll
        for (int k = 0; k < 3; ++k) rok = rok && to_q16(q[k], a.org[k], a.s, e16[k]);
        if (!rok) {
            if (slot == 0) {
                atomicExch(bad, 1);
                atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
            }
            continue;
        }
        Walk<T> w0;
        dda::walk_setup(w0, o16, e16);
        long long ne[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const long long dv = (long long)(e16[k] >> dda::kQShift) - (long long)(o16[k] >> dda::kQShift);
            ne[k] = dv < 0 ? -dv : dv;
        }
        const int A = (w0.ax >= w0.ay && w0.ax >= w0.az) ? 0 : (w0.ay >= w0.az ? 1 : 2);
        const long long pieces = ne[A] / kPieceEvents + 1;
        for (long long j = slot; j < pieces; j += kPieceSlots) {
            Walk<T> w = w0;
            long long s0 = 0, s1 = (long long)w0.n + 1;
            if (j > 0) {
                long long c[3];
                counts_after(w0, A, j * kPieceEvents, ne, c);
                s0 = c[0] + c[1] + c[2];
                w.qxy = (T)((long long)w0.qxy + c[0] * w0.ay - c[1] * w0.ax);
                w.qxz = (T)((long long)w0.qxz + c[0] * w0.az - c[2] * w0.ax);
                w.qyz = (T)((long long)w0.qyz + c[1] * w0.az - c[2] * w0.ay);
                w.vx = w0.vx + w0.sx * (int)c[0];
                w.vy = w0.vy + w0.sy * (int)c[1];
                w.vz = w0.vz + w0.sz * (int)c[2];
            }
            if (j + 1 < pieces) {
                long long c[3];
                counts_after(w0, A, (j + 1) * kPieceEvents, ne, c);
                s1 = c[0] + c[1] + c[2];
            }
            w.dX = w.dY = w.ndZ = 0;
            w.idx = 0;
            const long long last = w0.n;
            uint32_t prev_wi = 0xffffffffu, prev_bits = 0u;       // this thread's last OR (repeats skipped)
            for (long long s = s0; s < s1; ++s) {
                if ((unsigned)w.vx < (unsigned)a.nx && (unsigned)w.vy < (unsigned)a.ny &&
                    (unsigned)w.vz < (unsigned)a.nz) {
                    const uint32_t v = (uint32_t)w.vx + (uint32_t)a.nx * ((uint32_t)w.vy + (uint32_t)a.ny * (uint32_t)w.vz);
                    const uint32_t wi = v >> 2;
                    const uint32_t bits = (s == last ? hit : 1u) << ((v & 3u) * 8u);
                    const uint32_t have = wi == prev_wi ? prev_bits : 0u;
                    if ((have & bits) != bits) {
                        prev_wi = wi;
                        prev_bits = have | bits;
                        if (j == 0 && s < kDedupSteps) {          // near the sensor: one atomic per word per warp
                            const unsigned am = __activemask();
                            const unsigned peers = __match_any_sync(am, wi);
                            const uint32_t all = __reduce_or_sync(peers, bits);
                            if ((int)lane_id() == __ffs(peers) - 1) atomicOr(flags + wi, all);
                        } else {
                            atomicOr(flags + wi, bits);
                        }
                    }
                }
                dda::walk_step<T, kLayoutLinear, true>(w, mv);
            }
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

// Update pass, part 1: scan the flag bytes 16 at a time (a 256^3 grid is 16 MB of flags)
// and list every flagged voxel with its flags (one atomic per warp); the flags are cleared.
__global__ void __launch_bounds__(256) k_integrate_collect(uint4 *flags4, size_t n16, uint32_t *list,
                                                           uint32_t *ctl, const int *bad)
{
    const bool poisoned = *bad != 0;
    for (size_t i0 = blockIdx.x * (size_t)blockDim.x; i0 < n16; i0 += (size_t)gridDim.x * blockDim.x) {
        const size_t i = i0 + threadIdx.x;
        uint4 f4 = make_uint4(0u, 0u, 0u, 0u);
        if (i < n16) f4 = flags4[i];
        const bool any = (f4.x | f4.y | f4.z | f4.w) != 0u;
        if (any) flags4[i] = make_uint4(0u, 0u, 0u, 0u);
        const uint32_t fw[4] = {f4.x, f4.y, f4.z, f4.w};
        uint32_t cnt = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) cnt += __popc(__vcmpne4(fw[j], 0u)) >> 3;   // nonzero bytes
        if (poisoned) cnt = 0;
        // warp-wide exclusive prefix of cnt, one atomic per warp
        uint32_t pre = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, pre, o);
            if ((int)lane_id() >= o) pre += t;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
        uint32_t base = 0;
        if (lane_id() == 31 && tot) base = atomicAdd(ctl + kOccTouched, tot);
        base = __shfl_sync(0xffffffffu, base, 31) + pre - cnt;
        if (cnt == 0) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t rest = fw[j];
            while (rest) {
                const int b = (__ffs(rest) - 1) >> 3;
                const uint32_t f = (rest >> (8 * b)) & 0xffu;
                rest &= ~(0xffu << (8 * b));
                list[base++] = ((uint32_t)(16 * i) + 4u * j + (uint32_t)b) | ((f & 2u) << 30);   // bit 31: hit
            }
        }
    }
}

// Part 2: one thread per flagged voxel.  The map field is replaced by an AND then an OR on
// its word (no other thread writes this field, and one thread's atomics to one address
// stay ordered), so nothing waits on a read of the store.
__global__ void __launch_bounds__(256) k_integrate_apply(const uint32_t *__restrict__ list, const uint32_t *ctl_in,
                                                         float *L, ApplyArgs a, Geom g, uint32_t *words,
                                                         uint32_t *d_idx, uint16_t *d_val, uint32_t *n_deltas)
{
    const uint32_t n = ctl_in[kOccTouched];
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t e = list[t];
        const uint32_t v = e & 0x7fffffffu;
        const float l0 = L[v];
        const bool observed = !isnan(l0);
        float l1 = __fadd_rn(observed ? l0 : 0.0f, (e >> 31) ? a.lh : a.lm);
        l1 = fminf(fmaxf(l1, a.lo), a.hi);
        L[v] = l1;
        uint32_t c0 = 0, lv0 = 0, c1, lv1;
        if (observed) classify(l0, a, c0, lv0);
        classify(l1, a, c1, lv1);
        const bool changed = c0 != c1 || lv0 != lv1;
        if (changed && words) {
            const uint32_t x = v % (uint32_t)a.nx, r = v / (uint32_t)a.nx;
            const uint32_t y = r % (uint32_t)a.ny, z = r / (uint32_t)a.ny;
            const uint64_t pi = store_index(g, x, y, z);
            uint32_t *w = words + word_of(g, pi);
            const uint32_t sh = shift_of(g, pi);
            const uint32_t mask = g.vbits == 2 ? 3u : 0xffu;
            atomicAnd(w, ~(mask << sh));
            atomicOr(w, stored_value(g, c1, lv1) << sh);
        }
        const unsigned m = __ballot_sync(__activemask(), changed);
        if (!changed) continue;
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
        (st = o->runs.ensure((size_t)n * 5 + 16)) || (st = o->sorted.ensure((size_t)n * 24)) ||
        (st = o->filtered.ensure((size_t)n * 24)))
        return st;
    auto *keys = o->keys.as<unsigned long long>(), *keys_s = o->keys_alt.as<unsigned long long>();
    auto *idx = o->idx.as<uint32_t>(), *idx_s = o->idx_alt.as<uint32_t>();
    uint32_t *run_off = o->runs.as<uint32_t>(), *n_runs = run_off + n;
    uint8_t *head = reinterpret_cast<uint8_t *>(n_runs + 4);
    uint32_t *ctl = reinterpret_cast<uint32_t *>(o->d_ctl);
    const unsigned gr = grid_for(ctx, n, 256, 8);
    k_filter_keys<<<gr, 256, 0, ctx->stream>>>(d_pts, n, leaf, keys, idx, o->d_ctl + kOccBad, ctx->d_err);
    NBT_LAUNCHED(ctx);
    thrust::counting_iterator<uint32_t> iota(0);
    size_t t1 = 0, t2 = 0;
    NBT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys_s, idx, idx_s, (int)n, 0, kKeyBits, ctx->stream));
    NBT_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, iota, head, run_off, n_runs, (int)n, ctx->stream));
    const size_t tmp = t1 > t2 ? t1 : t2;
    if ((st = o->cub_tmp.ensure(tmp))) return st;
    size_t tt = tmp;
    NBT_CUDA(cub::DeviceRadixSort::SortPairs(o->cub_tmp.p, tt, keys, keys_s, idx, idx_s, (int)n, 0, kKeyBits,
                                             ctx->stream));
    k_filter_gather<<<gr, 256, 0, ctx->stream>>>(d_pts, idx_s, keys_s, n, o->sorted.as<double>(), head,
                                                 ctl + kOccValid);
    NBT_LAUNCHED(ctx);
    tt = tmp;
    NBT_CUDA(cub::DeviceSelect::Flagged(o->cub_tmp.p, tt, iota, head, run_off, n_runs, (int)n, ctx->stream));
    k_filter_centroid<<<grid_for(ctx, (size_t)n * kCentroidLanes, 256, 8), 256, 0, ctx->stream>>>(
        o->sorted.as<double>(), run_off, n_runs, ctl + kOccValid, o->filtered.as<double>(), d_count_out,
        ctl + kOccRays);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

// The hashed voxel filter of the integration path: o->filtered = the centroids (cells in
// the order of their first point, i.e. pixel order), ctl[kOccRays] = their number.
static nbt_status launch_voxel_filter_hashed(nbt_ctx ctx, nbt_occ_s *o, const double *d_pts, uint32_t n, double leaf)
{
    nbt_status st;
    int log2cap = 10;
    while ((1ull << log2cap) < 2ull * n) ++log2cap;
    const size_t cap = 1ull << log2cap;
    if ((st = o->hkeys.ensure(cap * 8)) || (st = o->hcount.ensure(cap * 16)) ||
        (st = o->cells.ensure((size_t)n * 5 + 16)) ||
        (st = o->idx.ensure((size_t)n * 4)) || (st = o->idx_alt.ensure((size_t)n * 4)) ||
        (st = o->sorted.ensure((size_t)n * 24)) || (st = o->filtered.ensure((size_t)n * 24)))
        return st;
    auto *table = o->hkeys.as<unsigned long long>();
    uint32_t *count = o->hcount.as<uint32_t>(), *fill = count + cap, *first_inv = fill + cap, *off = first_inv + cap;
    uint32_t *cells = o->cells.as<uint32_t>(), *n_cells = cells + n;
    uint8_t *head = reinterpret_cast<uint8_t *>(n_cells + 4);
    uint32_t *slot_of = o->idx.as<uint32_t>(), *seg = o->idx_alt.as<uint32_t>();
    uint32_t *ctl = reinterpret_cast<uint32_t *>(o->d_ctl);
    NBT_CUDA(cudaMemsetAsync(table, 0xff, cap * 8, ctx->stream));
    NBT_CUDA(cudaMemsetAsync(count, 0, cap * 12, ctx->stream));         // count, fill, first_inv
    const unsigned gr = grid_for(ctx, n, 256, 8);
    k_hash_insert<<<gr, 256, 0, ctx->stream>>>(d_pts, n, leaf, log2cap, table, count, first_inv, slot_of,
                                               o->d_ctl + kOccBad, ctx->d_err);
    NBT_LAUNCHED(ctx);
    size_t t1 = 0, t2 = 0;
    NBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, count, off, (int)cap, ctx->stream));
    NBT_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, slot_of, head, cells, n_cells, (int)n, ctx->stream));
    const size_t tmp = t1 > t2 ? t1 : t2;
    if ((st = o->cub_tmp.ensure(tmp))) return st;
    size_t tt = tmp;
    NBT_CUDA(cub::DeviceScan::ExclusiveSum(o->cub_tmp.p, tt, count, off, (int)cap, ctx->stream));
    k_hash_scatter<<<gr, 256, 0, ctx->stream>>>(slot_of, n, off, count, fill, seg);
    NBT_LAUNCHED(ctx);
    k_hash_place<<<gr, 256, 0, ctx->stream>>>(d_pts, slot_of, n, off, count, first_inv, seg,
                                              o->sorted.as<double>(), head);
    NBT_LAUNCHED(ctx);
    tt = tmp;
    NBT_CUDA(cub::DeviceSelect::Flagged(o->cub_tmp.p, tt, slot_of, head, cells, n_cells, (int)n, ctx->stream));
    k_hash_centroid<<<grid_for(ctx, (size_t)n * kCentroidLanes, 256, 8), 256, 0, ctx->stream>>>(
        o->sorted.as<double>(), d_pts, slot_of, n, cells, n_cells, off, count, first_inv, o->filtered.as<double>(),
        ctl + kOccRays);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_integrate(nbt_ctx ctx, nbt_occ_s *o, nbt_map m, const double sensor[3], const double *d_pts,
                            uint32_t n, const nbt_integrate_params &p)
{
    nbt_status st;
    ProfScope ps(ctx, NBT_KERNEL_INTEGRATE);
    // per-call control words: bad flag, ray count, voxels updated, delta count, valid points
    NBT_CUDA(cudaMemsetAsync(o->d_ctl, 0, kOccCtlInts * sizeof(int), ctx->stream));
    const double *rays = d_pts;
    const uint32_t *n_rays_dev = nullptr;      // filtered: the cell count is known on the device only
    o->last_points = n;
    o->last_filtered = p.leaf > 0.0;
    if (p.leaf > 0.0 && n > 0) {
        st = ctx->opt.filter_sort ? launch_voxel_filter(ctx, o, d_pts, n, p.leaf, nullptr)
                                  : launch_voxel_filter_hashed(ctx, o, d_pts, n, p.leaf);
        if (st) return st;
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
    if (n > 0) {
        const unsigned gr = grid_for(ctx, (size_t)n * kPieceSlots, kRayThreads, 8);
        if (wide)
            k_integrate_rays<long long><<<gr, kRayThreads, 0, ctx->stream>>>(rays, n_rays_dev, n, ra, o->d_flags,
                                                                     o->d_ctl + kOccBad, ctx->d_err);
        else
            k_integrate_rays<int><<<gr, kRayThreads, 0, ctx->stream>>>(rays, n_rays_dev, n, ra, o->d_flags,
                                                               o->d_ctl + kOccBad, ctx->d_err);
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
    const size_t n16 = (o->nvox + 15) / 16;
    k_integrate_collect<<<grid_for(ctx, n16, 256, 8), 256, 0, ctx->stream>>>(
        reinterpret_cast<uint4 *>(o->d_flags), n16, o->d_list, ctl, o->d_ctl + kOccBad);
    NBT_LAUNCHED(ctx);
    k_integrate_apply<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(o->d_list, ctl, o->d_L, aa, g, words, o->d_didx,
                                                                 o->d_dval, ctl + kOccDeltas);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
