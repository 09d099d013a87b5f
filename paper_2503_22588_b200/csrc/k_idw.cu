// IDW query over the ID ring buffer (Eq. 4).
//
//   G(x) = sum_u w_u * v_u(x),   v_u(x) = sum_j g_P,j d_j(x)^-p / sum_j d_j(x)^-p
//
// over the buffered clouds u = oldest..newest with w_u = 1/(m-u) (newest weighs 1,
// reading Q21), each cloud's own perspectives (Q20) and all of them (Q22); if the
// nearest perspective is closer than zero_eps, v_u is its gain (Q23).
//
//   k_idw_entry    grid (query blocks) x (entries): a block stages one entry's
//                  perspectives through shared memory; each thread holds 3 queries in
//                  registers and 16 lanes split the perspectives (interleaved; fp64
//                  partial sums combined by shuffles, so the result differs from a
//                  sequential sum only in rounding, < 1e-12 relative).  The nearest
//                  perspective is tracked on d^2 (monotone in d); only when it is within
//                  zero_eps is d = sqrt(d^2) evaluated and the lowest j among exactly
//                  equal d found by a rescan, so the zero-distance decision and the
//                  returned gain match the definition.
//   k_idw_combine  per query: G = sum_u w_u v_u in entry order (optionally / sum_u w_u).
#include "nbt_internal.cuh"

#ifndef NBT_IDW_EXACT_RCP
#define NBT_IDW_EXACT_RCP 0
#endif
#ifndef NBT_IDW_NR
#define NBT_IDW_NR 3              // refinement of the hardware reciprocal: 3 = one cubic step, 1/2 Newton steps
#endif
#ifndef NBT_IDW_HIMIN
#define NBT_IDW_HIMIN 1           // track min d^2 by its high word on the integer pipe
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
constexpr int kCombineBatch = 8;             // partial sums loaded together by the combines

// 1/x to within an ulp: the hardware approximation refined by one cubic step (the IEEE
// correctly-rounded __drcp_rn costs a longer sequence; IDW sums are compared with 1e-12
// relative tolerance, the zero-distance rule does not use it).  x = 0 gives +inf.
__device__ __forceinline__ double rcp_nr(double x)
{
#if NBT_IDW_EXACT_RCP
    return __drcp_rn(x);
#else
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    // rcp.approx is within 2^-20 (9.9e-7 measured, tools/rcp_probe.cu); with e = 1 - x r,
    // r (1 + e + e^2) has relative error e^3 (< 1e-18): one cubic step, 3 fma, replaces two
    // Newton steps (4 fma, error e^4); one Newton step alone leaves e^2 = 9.9e-13.
    double e = fma(-x, r, 1.0);
#if NBT_IDW_NR == 3
    e = fma(e, e, e);
    r = fma(r, e, r);
#else
    r = fma(r, e, r);
#if NBT_IDW_NR >= 2
    e = fma(-x, r, 1.0);
    r = fma(r, e, r);
#endif
#endif
    return r;
#endif
}

__device__ __forceinline__ double dist2(double x0, double x1, double x2, double p0, double p1, double p2)
{
    double dx = __dsub_rn(x0, p0), dy = __dsub_rn(x1, p1), dz = __dsub_rn(x2, p2);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Block (query block, entry e): 16 groups of kQPT (3) queries x 16 lanes.  The 16 lanes of a
// group split the entry's perspectives (interleaved), staged through shared memory; every
// perspective record a lane reads is used for its 3 queries (register blocking: one
// shared-memory read per 3 pairs), and the groups' partial sums combine by shuffles.  The
// weights use the fma-contracted d^2 (6 instead of 8 fp64 operations; its rounding is within
// the 1e-12 tolerance); only min d^2 is tracked per query and, when it may lie within zero_eps
// (1e-6 relative margin), the entry is rescanned with the correctly rounded d = sqrt(d^2) of the
// definition and the lowest j attaining the minimum decides the zero-distance rule exactly.
// The combine over the entries is fused: the last of a query block's `cap` blocks to finish
// (a counter per query block, reset by that block, so graph replays find it at zero) sums
// G = sum_u w_u v_u in entry order for its queries -- one launch per query call.
__device__ __forceinline__ double dist2_fast(double x0, double x1, double x2, double p0, double p1, double p2)
{
    const double dx = x0 - p0, dy = x1 - p1, dz = x2 - p2;
    return fma(dz, dz, fma(dy, dy, dx * dx));
}

#ifndef NBT_IDW_LB
#define NBT_IDW_LB 1              // resident blocks per SM the register allocation must allow
#endif
template <bool P2>        // power_p == 2 (the reciprocal) or a general power (pow)
__global__ void __launch_bounds__(kThreads, NBT_IDW_LB)
    k_idw_entry(const double *__restrict__ xyz, const double *__restrict__ gain, int32_t max_persp,
                const int32_t *__restrict__ meta, int32_t cap, const double *__restrict__ q, int32_t n_q,
                double power_p, double zero_eps, double *__restrict__ v_out, int *__restrict__ done,
                int32_t normalize, double *__restrict__ out)
{
    __shared__ double4 sp[kTile];
    __shared__ int last;
    const int e = blockIdx.y;
    const int pushes = meta[0];
    const int m = min(pushes, cap);
    if (e < m) {
        const int slot = (pushes - m + e) % cap;              // entry e, oldest first
        const int sub = threadIdx.x & (kSplit - 1);
        const int q0 = blockIdx.x * kQueries + (threadIdx.x / kSplit) * kQPT;
        const double *P = xyz + (size_t)slot * max_persp * 3;
        const double *G = gain + (size_t)slot * max_persp;
        const int np = meta[1 + slot];
        double x[kQPT][3];
#pragma unroll
        for (int k = 0; k < kQPT; ++k) {
            const int qi = min(q0 + k, n_q - 1);              // clamped: inactive queries compute garbage
            x[k][0] = q[3 * (size_t)qi]; x[k][1] = q[3 * (size_t)qi + 1]; x[k][2] = q[3 * (size_t)qi + 2];
        }
        const double hp = -0.5 * power_p;
        double num[kQPT], den[kQPT], d2min[kQPT];
        int hmin[kQPT];       // HIMIN: high word of min d^2 (d^2 >= 0, so its high word orders it)
#pragma unroll
        for (int k = 0; k < kQPT; ++k) {
            num[k] = 0.0; den[k] = 0.0; d2min[k] = __longlong_as_double(0x7ff0000000000000LL);
            hmin[k] = 0x7ff00000;
        }
        for (int base = 0; base < np; base += kTile) {
            const int nt = min(kTile, np - base);
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
                    if (NBT_IDW_HIMIN) hmin[k] = min(hmin[k], __double2hiint(d2));
                    else d2min[k] = fmin(d2min[k], d2);
                    const double w = P2 ? rcp_nr(d2) : pow(d2, hp);
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
                if (NBT_IDW_HIMIN) hmin[k] = min(hmin[k], __shfl_xor_sync(0xffffffffu, hmin[k], off));
                else d2min[k] = fmin(d2min[k], __shfl_xor_sync(0xffffffffu, d2min[k], off));
            }
        }
        // lane k of the group writes query k
        // (HIMIN: min d^2 rounded down to its high word, a lower bound, so the rescan test
        // below stays conservative)
        double nk = num[0], dk = den[0], mk = NBT_IDW_HIMIN ? __hiloint2double(hmin[0], 0) : d2min[0];
#pragma unroll
        for (int k = 1; k < kQPT; ++k)
            if (sub == k) { nk = num[k]; dk = den[k]; mk = NBT_IDW_HIMIN ? __hiloint2double(hmin[k], 0) : d2min[k]; }
        const int qi = q0 + sub;
        if (sub < kQPT && qi < n_q) {
            double v = nk / dk;
            const double lim = zero_eps * (1.0 + 1e-6);
            if (mk < lim * lim) {
                // the definition's nearest: correctly rounded d, lowest j among equal d
                const double y0 = q[3 * (size_t)qi], y1 = q[3 * (size_t)qi + 1], y2 = q[3 * (size_t)qi + 2];
                double dmin = __longlong_as_double(0x7ff0000000000000LL);
                int jmin = -1;
                for (int j = 0; j < np; ++j) {
                    const double d =
                        __dsqrt_rn(dist2(y0, y1, y2, P[3 * (size_t)j], P[3 * (size_t)j + 1], P[3 * (size_t)j + 2]));
                    if (d < dmin) { dmin = d; jmin = j; }
                }
                if (jmin >= 0 && dmin < zero_eps) v = G[jmin];
            }
            v_out[(size_t)e * n_q + qi] = v;
        }
    }
    if (!out) return;                                          // info cost: its own combine
    // fused combine: the last block of this query block sums the entries.  The barrier orders
    // the block's v_out stores before thread 0's fence (cumulative), so only thread 0 waits on it.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done + blockIdx.x, 1) == (int)gridDim.y - 1;
        if (last) done[blockIdx.x] = 0;                        // reset for the next call / graph replay
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int qi = blockIdx.x * kQueries + threadIdx.x; qi < min(n_q, (int)(blockIdx.x + 1) * kQueries);
         qi += kThreads) {
        double g = 0.0, wsum = 0.0;
        for (int u0 = 0; u0 < m; u0 += kCombineBatch) {
            // the batch's loads first (independent L2 reads), then the sum in entry order
            double vb[kCombineBatch];
#pragma unroll
            for (int t = 0; t < kCombineBatch; ++t)
                if (u0 + t < m) vb[t] = __ldcg(v_out + (size_t)(u0 + t) * n_q + qi);
#pragma unroll
            for (int t = 0; t < kCombineBatch; ++t) {
                if (u0 + t < m) {
                    const double wu = __ddiv_rn(1.0, (double)(m - u0 - t));
                    g = __dadd_rn(g, __dmul_rn(wu, vb[t]));
                    wsum = __dadd_rn(wsum, wu);
                }
            }
        }
        out[qi] = normalize ? __ddiv_rn(g, wsum) : g;
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

__global__ void k_idw_combine(const double *__restrict__ v, const int32_t *__restrict__ meta, int32_t cap, int32_t n_q,
                              int32_t normalize, double *__restrict__ out)
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
__global__ void k_info_cost(const double *__restrict__ v, const int32_t *__restrict__ meta, int32_t cap, InfoCostArgs a,
                            int32_t normalize, int *err)
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
            g = __dadd_rn(g, __dmul_rn(wu, v[(size_t)e * n_q + i]));
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
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_q * 8))) return st;
    dim3 grid((n_q + kQueries - 1) / kQueries, b->capacity);
    (power_p == 2.0 ? k_idw_entry<true> : k_idw_entry<false>)<<<grid, kThreads, 0, ctx->stream>>>(
        b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, a.pos, n_q, power_p, zero_eps,
        ctx->idw_tmp.as<double>(), nullptr, 0, nullptr);
    NBT_LAUNCHED(ctx);
    k_info_cost<<<(a.n_traj + 63) / 64, 64, 0, ctx->stream>>>(ctx->idw_tmp.as<double>(), b->d_meta, b->capacity, a,
                                                              normalize, ctx->d_err);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_idw(nbt_ctx ctx, const nbt_idbuf_s *b, const double *d_q, int32_t n_q, double power_p,
                      double zero_eps, int32_t normalize, double *d_out, int32_t knn)
{
    if (n_q == 0) return NBT_OK;
    nbt_status st;
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_q * 8))) return st;
    if (knn > 0) {
        const long long warps = (long long)n_q * b->capacity;
        k_idw_entry_knn<<<(unsigned)((warps + 7) / 8), 256, 0, ctx->stream>>>(
            b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, d_q, n_q, power_p, zero_eps, knn,
            ctx->idw_tmp.as<double>());
        NBT_LAUNCHED(ctx);
        k_idw_combine<<<(n_q + 127) / 128, 128, 0, ctx->stream>>>(ctx->idw_tmp.as<double>(), b->d_meta, b->capacity,
                                                                   n_q, normalize, d_out);
        NBT_LAUNCHED(ctx);
        return NBT_OK;
    }
    // per-query-block completion counters in their own buffer, zero between calls (the last
    // block of a query block resets its counter); zeroed once when (re)allocated
    const int nqb = (n_q + kQueries - 1) / kQueries;
    if ((st = ctx->idw_done.ensure((size_t)nqb * 4))) return st;
    int *done = ctx->idw_done.as<int>();
    if (ctx->idw_done_at != (void *)done || ctx->idw_done_zeroed < (size_t)nqb) {
        NBT_CUDA(cudaMemsetAsync(done, 0, ctx->idw_done.cap, ctx->stream));
        ctx->idw_done_zeroed = ctx->idw_done.cap / 4;
        ctx->idw_done_at = done;
    }
    dim3 grid(nqb, b->capacity);
    (power_p == 2.0 ? k_idw_entry<true> : k_idw_entry<false>)<<<grid, kThreads, 0, ctx->stream>>>(
        b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, d_q, n_q, power_p, zero_eps,
        ctx->idw_tmp.as<double>(), done, normalize, d_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
