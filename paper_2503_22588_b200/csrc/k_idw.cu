// IDW query over the ID ring buffer (Eq. 4).
//
//   G(x) = sum_u w_u * v_u(x),   v_u(x) = sum_j g_P,j d_j(x)^-p / sum_j d_j(x)^-p
//
// over the buffered clouds u = oldest..newest with w_u = 1/(m-u) (newest weighs 1,
// reading Q21), each cloud's own perspectives (Q20) and all of them (Q22); if the
// nearest perspective is closer than zero_eps, v_u is its gain (Q23).
//
//   k_idw_entry    grid (query blocks) x (entries) x (perspective chunks): a block stages
//                  one chunk of an entry's perspectives through shared memory; each thread
//                  holds 3 queries in registers and 16 lanes split the chunk (interleaved;
//                  fp64 partial sums combined by shuffles) and writes the chunk's partial
//                  (sum g w, sum w, min d^2) per query.  The result differs from a
//                  sequential sum only in rounding (< 1e-12 relative).
//   k_idw_combine  per query: per entry the chunk partials in order -> v_u (the zero-
//                  distance rule decided exactly: when the nearest perspective may be
//                  within zero_eps the entry is rescanned with the correctly rounded d and
//                  the lowest j among exactly equal d wins, as in the definition), then
//                  G = sum_u w_u v_u in entry order (optionally / sum_u w_u).
#include "nbt_internal.cuh"

#ifndef NBT_IDW_EXACT_RCP
#define NBT_IDW_EXACT_RCP 0
#endif

namespace nbt {
namespace {

#ifndef NBT_IDW_QPT
#define NBT_IDW_QPT 3
#endif
#ifndef NBT_IDW_SPLIT
#define NBT_IDW_SPLIT 16
#endif
constexpr int kQPT = NBT_IDW_QPT;            // queries per thread (register-blocked)
constexpr int kSplit = NBT_IDW_SPLIT;        // lanes sharing one (query group, entry)
constexpr int kGroups = 256 / kSplit;        // query groups per block
constexpr int kThreads = kGroups * kSplit;   // 256
constexpr int kQueries = kGroups * kQPT;     // 48 queries per block
constexpr int kTile = 512;

// 1/x to within an ulp: the hardware approximation refined by two Newton steps (the IEEE
// correctly-rounded __drcp_rn costs a longer sequence; IDW sums are compared with 1e-12
// relative tolerance, the zero-distance rule does not use it).  x = 0 gives +inf.
__device__ __forceinline__ double rcp_nr(double x)
{
#if NBT_IDW_EXACT_RCP
    return __drcp_rn(x);
#else
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
#endif
}

__device__ __forceinline__ double dist2(double x0, double x1, double x2, double p0, double p1, double p2)
{
    double dx = __dsub_rn(x0, p0), dy = __dsub_rn(x1, p1), dz = __dsub_rn(x2, p2);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Block (query block, entry e, perspective chunk c): 16 groups of kQPT (3) queries x 16
// lanes.  The 16 lanes of a group split the chunk's perspectives (interleaved), staged
// through shared memory; every perspective record a lane reads is used for its 3 queries
// (register blocking), and the groups' partial sums combine by shuffles.  The chunk's
// partial (sum g w, sum w, min d^2) per query goes to part[e][c][q]; k_idw_combine adds
// the chunks in order.  Splitting an entry's perspectives over chunks gives the launch
// enough blocks to fill every SM (1984 queries x 10 entries is only 420 blocks of 48
// queries, ~1.4 waves at 2 blocks per SM, the tail SM-idle).  w = 1/d^2 on the fma-
// contracted d^2 (its rounding is within the 1e-12 tolerance); min d^2 of the contracted
// form only triggers the zero-distance rule, which k_idw_combine decides exactly.
struct IdwPart { double num, den, d2min; };

__device__ __forceinline__ double dist2_fast(double x0, double x1, double x2, double p0, double p1, double p2)
{
    const double dx = x0 - p0, dy = x1 - p1, dz = x2 - p2;
    return fma(dz, dz, fma(dy, dy, dx * dx));
}

#ifndef NBT_IDW_LB
#define NBT_IDW_LB 1              // resident blocks per SM the register allocation must allow
#endif
__global__ void __launch_bounds__(kThreads, NBT_IDW_LB)
    k_idw_entry(const double *__restrict__ xyz, const double *__restrict__ gain, int32_t max_persp,
                const int32_t *__restrict__ meta, int32_t cap, const double *__restrict__ q, int32_t n_q,
                double power_p, int32_t chunk, int32_t n_chunks, IdwPart *__restrict__ part)
{
    __shared__ double4 sp[kTile];
    // persistent: units (query block, entry, chunk), chunk-major then entry, dealt round-robin
    const int nqb = (n_q + kQueries - 1) / kQueries;
    const int units = nqb * cap * n_chunks;
    const int pushes = meta[0];
    const int m = min(pushes, cap);
    const int sub = threadIdx.x & (kSplit - 1);
    const bool p2 = power_p == 2.0;
    const double hp = -0.5 * power_p;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int qb = u % nqb;
        const int e = (u / nqb) % cap;
        const int c = u / (nqb * cap);
        if (e >= m) continue;                                 // block-uniform
        const int slot = (pushes - m + e) % cap;              // entry e, oldest first
        const int q0 = qb * kQueries + (threadIdx.x / kSplit) * kQPT;
        const double *P = xyz + (size_t)slot * max_persp * 3;
        const double *G = gain + (size_t)slot * max_persp;
        const int np = meta[1 + slot];
        const int j0 = c * chunk, j1 = min(np, j0 + chunk);
        double x[kQPT][3];
#pragma unroll
        for (int k = 0; k < kQPT; ++k) {
            const int qi = min(q0 + k, n_q - 1);              // clamped: inactive queries compute garbage
            x[k][0] = q[3 * (size_t)qi]; x[k][1] = q[3 * (size_t)qi + 1]; x[k][2] = q[3 * (size_t)qi + 2];
        }
        double num[kQPT], den[kQPT], d2min[kQPT];
#pragma unroll
        for (int k = 0; k < kQPT; ++k) {
            num[k] = 0.0; den[k] = 0.0; d2min[k] = __longlong_as_double(0x7ff0000000000000LL);
        }
        for (int base = j0; base < j1; base += kTile) {
            const int nt = min(kTile, j1 - base);
            __syncthreads();
            for (int t = threadIdx.x; t < nt; t += kThreads)
                sp[t] = make_double4(P[3 * (size_t)(base + t)], P[3 * (size_t)(base + t) + 1],
                                     P[3 * (size_t)(base + t) + 2], G[base + t]);
            __syncthreads();
#pragma unroll 2
            for (int t = sub; t < nt; t += kSplit) {
                const double4 r = sp[t];
#pragma unroll
                for (int k = 0; k < kQPT; ++k) {
                    const double d2 = dist2_fast(x[k][0], x[k][1], x[k][2], r.x, r.y, r.z);
                    d2min[k] = fmin(d2min[k], d2);
                    const double w = p2 ? rcp_nr(d2) : pow(d2, hp);
                    num[k] = fma(r.w, w, num[k]);
                    den[k] += w;
                }
            }
        }
#pragma unroll
        for (int off = kSplit / 2; off > 0; off >>= 1) {
#pragma unroll
            for (int k = 0; k < kQPT; ++k) {
                num[k] += __shfl_xor_sync(0xffffffffu, num[k], off);
                den[k] += __shfl_xor_sync(0xffffffffu, den[k], off);
                d2min[k] = fmin(d2min[k], __shfl_xor_sync(0xffffffffu, d2min[k], off));
            }
        }
        // lane k of the group writes query k
        double nk = num[0], dk = den[0], mk = d2min[0];
#pragma unroll
        for (int k = 1; k < kQPT; ++k)
            if (sub == k) { nk = num[k]; dk = den[k]; mk = d2min[k]; }
        const int qi = q0 + sub;
        if (sub < kQPT && qi < n_q) part[((size_t)e * n_chunks + c) * n_q + qi] = IdwPart{nk, dk, mk};
    }
}

// Optional k-nearest Eq. 4 (reading Q22): one warp per (query, entry).  Every lane keeps the
// 16 nearest of its perspectives (j = lane, lane + 32, ...) sorted by (d^2, j) in registers;
// knn rounds of a warp-wide (d^2, j) argmin then take the k nearest of the entry, each
// summed by the lane that holds it (the order differs from the oracle's ascending j only in
// rounding).  The zero-distance rule is the same as k_idw_entry's.
constexpr int kKnnMax = 16;

__device__ __forceinline__ bool dj_less(double a, int ja, double b, int jb)
{
    return a < b || (a == b && ja < jb);
}

__global__ void __launch_bounds__(256)
    k_idw_entry_knn(const double *__restrict__ xyz, const double *__restrict__ gain, int32_t max_persp,
                    const int32_t *__restrict__ meta, int32_t cap, const double *__restrict__ q, int32_t n_q,
                    double power_p, double zero_eps, int32_t knn, double *__restrict__ v_out)
{
    const int lane = threadIdx.x & 31;
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int pushes = meta[0];
    const int m = min(pushes, cap);
    const int e = (int)(gw / n_q);
    const int qi = (int)(gw % n_q);
    if (e >= m) return;
    const int slot = (pushes - m + e) % cap;
    const double *P = xyz + (size_t)slot * max_persp * 3;
    const double *G = gain + (size_t)slot * max_persp;
    const int np = meta[1 + slot];
    const double x0 = q[3 * (size_t)qi], x1 = q[3 * (size_t)qi + 1], x2 = q[3 * (size_t)qi + 2];
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double d[kKnnMax];
    int jj[kKnnMax];
#pragma unroll
    for (int t = 0; t < kKnnMax; ++t) { d[t] = inf; jj[t] = 0x7fffffff; }
    double d2min = inf;
    for (int j = lane; j < np; j += 32) {
        const double d2 = dist2(x0, x1, x2, P[3 * (size_t)j], P[3 * (size_t)j + 1], P[3 * (size_t)j + 2]);
        d2min = fmin(d2min, d2);
        if (dj_less(d2, j, d[kKnnMax - 1], jj[kKnnMax - 1])) {
            d[kKnnMax - 1] = d2;
            jj[kKnnMax - 1] = j;
#pragma unroll
            for (int t = kKnnMax - 1; t > 0; --t) {
                if (dj_less(d[t], jj[t], d[t - 1], jj[t - 1])) {
                    const double td = d[t]; d[t] = d[t - 1]; d[t - 1] = td;
                    const int tj = jj[t]; jj[t] = jj[t - 1]; jj[t - 1] = tj;
                }
            }
        }
    }
    const bool p2 = power_p == 2.0;
    const double hp = -0.5 * power_p;
    double num = 0.0, den = 0.0;
    for (int r = 0; r < knn; ++r) {
        double bd = d[0];
        int bj = jj[0];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, off);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
            if (dj_less(od, oj, bd, bj)) { bd = od; bj = oj; }
        }
        if (bj == 0x7fffffff) break;                  // fewer than knn perspectives
        if (jj[0] == bj) {                            // this lane holds the winner
            const double w = p2 ? rcp_nr(bd) : pow(bd, hp);
            num = fma(G[bj], w, num);
            den += w;
#pragma unroll
            for (int t = 0; t < kKnnMax - 1; ++t) { d[t] = d[t + 1]; jj[t] = jj[t + 1]; }
            d[kKnnMax - 1] = inf;
            jj[kKnnMax - 1] = 0x7fffffff;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
        d2min = fmin(d2min, __shfl_xor_sync(0xffffffffu, d2min, off));
    }
    if (lane != 0) return;
    double v = num / den;
    const double dmin = __dsqrt_rn(d2min);
    if (dmin < zero_eps) {
        for (int j = 0; j < np; ++j) {
            const double d2 = dist2(x0, x1, x2, P[3 * (size_t)j], P[3 * (size_t)j + 1], P[3 * (size_t)j + 2]);
            if (__dsqrt_rn(d2) == dmin) { v = G[j]; break; }
        }
    }
    v_out[(size_t)e * n_q + qi] = v;
}

// v_e(x) of entry e from its chunk partials, with the zero-distance rule (Q23) decided
// exactly: if the nearest perspective may be closer than zero_eps (by the contracted min d^2,
// with a 1e-6 relative margin), the entry is rescanned with the correctly rounded d =
// sqrt(d^2) of the definition, and the lowest j attaining the minimum gives v_e when that
// minimum is < zero_eps.  Chunk sums are added in chunk order (one lane) so the value does
// not depend on the launch shape beyond the chunking.
__device__ double idw_entry_value(double num, double den, double d2m, int e, const double *xyz, const double *gain,
                                  int32_t max_persp, const int32_t *meta, int32_t cap, const double *q, int qi,
                                  double zero_eps)
{
    double v = num / den;
    const double lim = zero_eps * (1.0 + 1e-6);
    if (d2m < lim * lim) {
        const int pushes = meta[0];
        const int m = min(pushes, cap);
        const int slot = (pushes - m + e) % cap;
        const double *P = xyz + (size_t)slot * max_persp * 3;
        const int np = meta[1 + slot];
        const double y0 = q[3 * (size_t)qi], y1 = q[3 * (size_t)qi + 1], y2 = q[3 * (size_t)qi + 2];
        double dmin = __longlong_as_double(0x7ff0000000000000LL);
        int jmin = -1;
        for (int j = 0; j < np; ++j) {
            const double d = __dsqrt_rn(dist2(y0, y1, y2, P[3 * (size_t)j], P[3 * (size_t)j + 1], P[3 * (size_t)j + 2]));
            if (d < dmin) { dmin = d; jmin = j; }
        }
        if (jmin >= 0 && dmin < zero_eps) v = gain[(size_t)slot * max_persp + jmin];
    }
    return v;
}

// Per-entry values of one query, one warp: lane e (< m) adds entry e's chunk partials in
// order and applies the zero-distance rule; returns v_e on lane e.
__device__ __forceinline__ double idw_chunked_entry_value(const IdwPart *part, int e, int n_chunks, int n_q, int qi,
                                                          const double *xyz, const double *gain, int32_t max_persp,
                                                          const int32_t *meta, int32_t cap, const double *q,
                                                          double zero_eps)
{
    double num = 0.0, den = 0.0, d2m = __longlong_as_double(0x7ff0000000000000LL);
    for (int c = 0; c < n_chunks; ++c) {
        const IdwPart p = part[((size_t)e * n_chunks + c) * n_q + qi];
        num += p.num;
        den += p.den;
        d2m = fmin(d2m, p.d2min);
    }
    return idw_entry_value(num, den, d2m, e, xyz, gain, max_persp, meta, cap, q, qi, zero_eps);
}

// One warp per query: the entries' values in parallel (lanes), then G = sum_u w_u v_u in entry
// order on lane 0 (optionally / sum_u w_u).  cap <= 32 (nbt_idbuf_create allows 64: larger
// rings loop over lanes).
__global__ void k_idw_combine(const IdwPart *__restrict__ part, int32_t n_chunks, const double *__restrict__ xyz,
                              const double *__restrict__ gain, int32_t max_persp, const int32_t *__restrict__ meta,
                              int32_t cap, const double *__restrict__ q, int32_t n_q, double zero_eps,
                              int32_t normalize, double *__restrict__ out)
{
    const int lane = threadIdx.x & 31;
    const int qi = (int)(((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (qi >= n_q) return;
    const int m = min(meta[0], cap);
    double g = 0.0, wsum = 0.0;
    for (int e0 = 0; e0 < m; e0 += 32) {
        const double v = e0 + lane < m ? idw_chunked_entry_value(part, e0 + lane, n_chunks, n_q, qi, xyz, gain,
                                                                 max_persp, meta, cap, q, zero_eps)
                                       : 0.0;
        for (int e = e0; e < min(m, e0 + 32); ++e) {
            const double ve = __shfl_sync(0xffffffffu, v, e - e0);
            const double wu = __ddiv_rn(1.0, (double)(m - e));
            g = __dadd_rn(g, __dmul_rn(wu, ve));
            wsum = __dadd_rn(wsum, wu);
        }
    }
    if (lane == 0) out[qi] = normalize ? __ddiv_rn(g, wsum) : g;
}

// Combine of per-entry values (the k-nearest path writes v_e directly).
__global__ void k_idw_combine_values(const double *__restrict__ v, const int32_t *__restrict__ meta, int32_t cap,
                                     int32_t n_q, int32_t normalize, double *__restrict__ out)
{
    const int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= n_q) return;
    const int m = min(meta[0], cap);
    double g = 0.0, wsum = 0.0;
    for (int e = 0; e < m; ++e) {
        const double wu = __ddiv_rn(1.0, (double)(m - e));
        g = __dadd_rn(g, __dmul_rn(wu, v[(size_t)e * n_q + qi]));
        wsum = __dadd_rn(wsum, wu);
    }
    out[qi] = normalize ? __ddiv_rn(g, wsum) : g;
}

// Information cost (f2): one thread per trajectory, poses in order.  O by the rounded-
// once dot product / norms (the same expression as the definition, so the FoV decision
// is reproducible), G from the per-entry IDW values, c = sum_k w_i / (O G + eps).
__global__ void k_info_cost(const IdwPart *__restrict__ part, int32_t n_chunks, const double *__restrict__ xyz,
                            const double *__restrict__ gain, int32_t max_persp, const int32_t *__restrict__ meta,
                            int32_t cap, double zero_eps, InfoCostArgs a, int32_t normalize, int *err)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n_traj) return;
    const int m = min(meta[0], cap);
    const int n_q = a.n_traj * a.per;
    double c = 0.0;
    for (int k = 0; k < a.per; ++k) {
        const int i = t * a.per + k;
        double g = 0.0, wsum = 0.0;
        for (int e = 0; e < m; ++e) {
            const double wu = __ddiv_rn(1.0, (double)(m - e));
            const double v = idw_chunked_entry_value(part, e, n_chunks, n_q, i, xyz, gain, max_persp, meta, cap, a.pos,
                                                     zero_eps);
            g = __dadd_rn(g, __dmul_rn(wu, v));
            wsum = __dadd_rn(wsum, wu);
        }
        if (normalize) g = __ddiv_rn(g, wsum);
        const double *p = a.pos + 3 * (size_t)i, *ax = a.axis + 3 * (size_t)i;
        const double d0 = __dsub_rn(a.poi[0], p[0]), d1 = __dsub_rn(a.poi[1], p[1]), d2 = __dsub_rn(a.poi[2], p[2]);
        const double nd = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
        const double na =
            __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ax[0], ax[0]), __dmul_rn(ax[1], ax[1])), __dmul_rn(ax[2], ax[2])));
        double o;
        if (nd < 1e-9 || !(na > 0.0)) {
            atomicCAS(err, 0, nd < 1e-9 ? (int)NBT_ERR_DEGENERATE : (int)NBT_ERR_INVALID_ARG);
            o = __longlong_as_double(0x7ff8000000000000LL);
        } else {
            const double dot = __dadd_rn(__dadd_rn(__dmul_rn(ax[0], d0), __dmul_rn(ax[1], d1)), __dmul_rn(ax[2], d2));
            const double cs = __ddiv_rn(dot, __dmul_rn(na, nd));
            o = cs >= a.cos_cut ? cs : 0.0;
        }
        if (a.o_out) a.o_out[i] = o;
        if (a.g_out) a.g_out[i] = g;
        c = __dadd_rn(c, __ddiv_rn(a.w_i, __dadd_rn(__dmul_rn(o, g), a.eps)));
    }
    a.c_out[t] = c;
}

// Ring push, device side (so a captured CUDA graph can replay it): copy the cloud into
// slot pushes % cap, then advance the counter in a second, single-thread kernel.
__global__ void k_idbuf_copy(const int32_t *__restrict__ meta, int32_t cap, int32_t max_persp,
                             const double *__restrict__ src_xyz, const double *__restrict__ src_gain, int32_t n,
                             double *__restrict__ xyz, double *__restrict__ gain)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 4 * n) return;
    const int slot = meta[0] % cap;
    if (i < 3 * n) xyz[(size_t)slot * max_persp * 3 + i] = src_xyz[i];
    else gain[(size_t)slot * max_persp + (i - 3 * n)] = src_gain[i - 3 * n];
}

__global__ void k_idbuf_advance(int32_t *meta, int32_t cap, int32_t n)
{
    const int slot = meta[0] % cap;
    meta[1 + slot] = n;
    meta[0] = meta[0] + 1;
}

// Small clouds: copy and advance in one single-block launch (every thread reads the slot
// before the barrier, thread 0 advances the ring after it).
constexpr int kPushOneBlock = 1024;
__global__ void __launch_bounds__(kPushOneBlock) k_idbuf_push_small(int32_t *meta, int32_t cap, int32_t max_persp,
                                                                    const double *__restrict__ src_xyz,
                                                                    const double *__restrict__ src_gain, int32_t n,
                                                                    double *__restrict__ xyz, double *__restrict__ gain)
{
    const int slot = meta[0] % cap;
    for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) {
        if (i < 3 * n) xyz[(size_t)slot * max_persp * 3 + i] = src_xyz[i];
        else gain[(size_t)slot * max_persp + (i - 3 * n)] = src_gain[i - 3 * n];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        meta[1 + slot] = n;
        meta[0] = meta[0] + 1;
    }
}

#ifndef NBT_IDW_MIN_BLOCKS
#define NBT_IDW_MIN_BLOCKS 4      // units per resident block slot the chunking aims for (balance of the persistent grid)
#endif
#ifndef NBT_IDW_CHUNK_MIN
#define NBT_IDW_CHUNK_MIN 64
#endif
// Perspective chunk per block: enough (query block, entry, chunk) blocks for ~NBT_IDW_MIN_BLOCKS
// per SM, chunks a multiple of 32 and at least NBT_IDW_CHUNK_MIN perspectives.
int idw_blocks_per_sm()
{
    static int bps = [] {
        int v = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_idw_entry, kThreads, 0);
        return v > 0 ? v : 1;
    }();
    return bps;
}

// Persistent grid of the entry kernel: every resident block slot, at most one per unit.
int idw_grid(nbt_ctx ctx, const nbt_idbuf_s *b, int32_t n_q, int32_t n_chunks)
{
    const long long units = (long long)((n_q + kQueries - 1) / kQueries) * b->capacity * n_chunks;
    const long long slots = (long long)ctx->num_sms * idw_blocks_per_sm();
    return (int)(units < slots ? units : slots);
}

void idw_chunks(nbt_ctx ctx, const nbt_idbuf_s *b, int32_t n_q, int32_t &chunk, int32_t &n_chunks)
{
    const long long base = (long long)((n_q + kQueries - 1) / kQueries) * b->capacity;
    const long long want = (long long)ctx->num_sms * idw_blocks_per_sm() * NBT_IDW_MIN_BLOCKS;
    long long s = (want + base - 1) / base;
    long long c = ((long long)b->max_persp + s - 1) / s;
    c = (c + 31) / 32 * 32;
    if (c < NBT_IDW_CHUNK_MIN) c = NBT_IDW_CHUNK_MIN;
    chunk = (int32_t)c;
    n_chunks = (int32_t)((b->max_persp + c - 1) / c);
}

}  // namespace

nbt_status launch_idbuf_push(nbt_ctx ctx, nbt_idbuf_s *b, const double *d_xyz, const double *d_gain, int32_t n)
{
    if (4 * n <= 8 * kPushOneBlock) {
        k_idbuf_push_small<<<1, kPushOneBlock, 0, ctx->stream>>>(b->d_meta, b->capacity, b->max_persp, d_xyz, d_gain,
                                                                 n, b->d_xyz, b->d_gain);
        NBT_LAUNCHED(ctx);
        return NBT_OK;
    }
    k_idbuf_copy<<<(4 * n + 255) / 256, 256, 0, ctx->stream>>>(b->d_meta, b->capacity, b->max_persp, d_xyz, d_gain,
                                                                  n, b->d_xyz, b->d_gain);
    NBT_LAUNCHED(ctx);
    k_idbuf_advance<<<1, 1, 0, ctx->stream>>>(b->d_meta, b->capacity, n);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_info_cost(nbt_ctx ctx, const nbt_idbuf_s *b, const InfoCostArgs &a, double power_p,
                            double zero_eps, int32_t normalize)
{
    const int32_t n_q = a.n_traj * a.per;
    if (n_q == 0) return NBT_OK;
    nbt_status st;
    int32_t chunk, n_chunks;
    idw_chunks(ctx, b, n_q, chunk, n_chunks);
    if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_chunks * n_q * sizeof(IdwPart)))) return st;
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    IdwPart *part = ctx->idw_tmp.as<IdwPart>();
    k_idw_entry<<<idw_grid(ctx, b, n_q, n_chunks), kThreads, 0, ctx->stream>>>(
        b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, a.pos, n_q, power_p, chunk, n_chunks, part);
    NBT_LAUNCHED(ctx);
    k_info_cost<<<(a.n_traj + 63) / 64, 64, 0, ctx->stream>>>(part, n_chunks, b->d_xyz, b->d_gain, b->max_persp,
                                                              b->d_meta, b->capacity, zero_eps, a, normalize,
                                                              ctx->d_err);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_idw(nbt_ctx ctx, const nbt_idbuf_s *b, const double *d_q, int32_t n_q, double power_p,
                      double zero_eps, int32_t normalize, double *d_out, int32_t knn)
{
    if (n_q == 0) return NBT_OK;
    nbt_status st;
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    if (knn > 0) {
        if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_q * 8))) return st;
        const long long warps = (long long)n_q * b->capacity;
        k_idw_entry_knn<<<(unsigned)((warps + 7) / 8), 256, 0, ctx->stream>>>(
            b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, d_q, n_q, power_p, zero_eps, knn,
            ctx->idw_tmp.as<double>());
        NBT_LAUNCHED(ctx);
        k_idw_combine_values<<<(n_q + 127) / 128, 128, 0, ctx->stream>>>(ctx->idw_tmp.as<double>(), b->d_meta,
                                                                          b->capacity, n_q, normalize, d_out);
        NBT_LAUNCHED(ctx);
        return NBT_OK;
    }
    int32_t chunk, n_chunks;
    idw_chunks(ctx, b, n_q, chunk, n_chunks);
    if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_chunks * n_q * sizeof(IdwPart)))) return st;
    IdwPart *part = ctx->idw_tmp.as<IdwPart>();
    k_idw_entry<<<idw_grid(ctx, b, n_q, n_chunks), kThreads, 0, ctx->stream>>>(
        b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, d_q, n_q, power_p, chunk, n_chunks, part);
    NBT_LAUNCHED(ctx);
    k_idw_combine<<<(unsigned)(((size_t)n_q * 32 + 255) / 256), 256, 0, ctx->stream>>>(part, n_chunks, b->d_xyz, b->d_gain, b->max_persp,
                                                               b->d_meta, b->capacity, d_q, n_q, zero_eps, normalize,
                                                               d_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
