// IDW query over the ID ring buffer (Eq. 4).
//
//   G(x) = sum_u w_u * v_u(x),   v_u(x) = sum_j g_P,j d_j(x)^-p / sum_j d_j(x)^-p
//
// over the buffered clouds u = oldest..newest with w_u = 1/(m-u) (newest weighs 1,
// reading Q21), each cloud's own perspectives (Q20) and all of them (Q22); if the
// nearest perspective is closer than zero_eps, v_u is its gain (Q23).
//
//   k_idw_entry    grid (query blocks) x (entries): a block stages one entry's
//                  perspectives through shared memory; 8 lanes per query split them
//                  (interleaved; fp64 partial sums combined by shuffles, so the
//                  result differs from a sequential sum only in rounding, < 1e-12
//                  relative).  The nearest perspective is tracked on d^2 (monotone in
//                  d); only when it is within zero_eps is d = sqrt(d^2) evaluated, with a
//                  second pass to pick the lowest j among exactly equal d, so the
//                  zero-distance decision and the returned gain match the definition.
//   k_idw_combine  per query: G = sum_u w_u v_u in entry order (optionally / sum_u w_u).
#include "nbt_internal.cuh"

namespace nbt {
namespace {

constexpr int kQueries = 32;     // queries per block
constexpr int kSplit = 8;        // lanes sharing one (query, entry)
constexpr int kThreads = kQueries * kSplit;
constexpr int kTile = 512;

__device__ __forceinline__ double dist2(double x0, double x1, double x2, double p0, double p1, double p2)
{
    double dx = __dsub_rn(x0, p0), dy = __dsub_rn(x1, p1), dz = __dsub_rn(x2, p2);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Block (query block, entry e): 32 queries x 8 lanes each; the 8 lanes of a query split
// the entry's perspectives (interleaved), staged through shared memory, and
// combine (sum of num, sum of den, argmin of d^2 with lowest j) by warp shuffles.
__global__ void __launch_bounds__(kThreads)
    k_idw_entry(const double *__restrict__ xyz, const double *__restrict__ gain, int32_t max_persp,
                const int32_t *__restrict__ meta, int32_t cap, const double *__restrict__ q, int32_t n_q,
                double power_p, double zero_eps, double *__restrict__ v_out)
{
    __shared__ double sp[kTile][4];
    const int e = blockIdx.y;
    const int pushes = meta[0];
    const int m = min(pushes, cap);
    if (e >= m) return;
    const int slot = (pushes - m + e) % cap;                  // entry e, oldest first
    const int sub = threadIdx.x & (kSplit - 1);
    const int qi = blockIdx.x * kQueries + (threadIdx.x / kSplit);
    const bool active = qi < n_q;
    const double *P = xyz + (size_t)slot * max_persp * 3;
    const double *G = gain + (size_t)slot * max_persp;
    const int np = meta[1 + slot];
    double x0 = 0.0, x1 = 0.0, x2 = 0.0;
    if (active) { x0 = q[3 * (size_t)qi]; x1 = q[3 * (size_t)qi + 1]; x2 = q[3 * (size_t)qi + 2]; }
    const bool p2 = power_p == 2.0;
    const double hp = -0.5 * power_p;
    double num = 0.0, den = 0.0, d2min = __longlong_as_double(0x7ff0000000000000LL);
    int jmin = 0x7fffffff;
    for (int base = 0; base < np; base += kTile) {
        const int nt = min(kTile, np - base);
        __syncthreads();
        for (int t = threadIdx.x; t < nt; t += kThreads) {
            sp[t][0] = P[3 * (size_t)(base + t)];
            sp[t][1] = P[3 * (size_t)(base + t) + 1];
            sp[t][2] = P[3 * (size_t)(base + t) + 2];
            sp[t][3] = G[base + t];
        }
        __syncthreads();
        // sub-lane s takes t = s, s+8, ...: the 8 lanes of a query read 8 consecutive
        // 32-byte records (no shared-memory bank conflicts)
#pragma unroll 4
        for (int t = sub; t < nt; t += kSplit) {
            const double d2 = dist2(x0, x1, x2, sp[t][0], sp[t][1], sp[t][2]);
            if (d2 < d2min) { d2min = d2; jmin = base + t; }
            const double w = p2 ? __drcp_rn(d2) : pow(d2, hp);
            num = fma(sp[t][3], w, num);
            den += w;
        }
    }
#pragma unroll
    for (int off = kSplit / 2; off > 0; off >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, off);
        den += __shfl_xor_sync(0xffffffffu, den, off);
        const double od = __shfl_xor_sync(0xffffffffu, d2min, off);
        const int oj = __shfl_xor_sync(0xffffffffu, jmin, off);
        if (od < d2min || (od == d2min && oj < jmin)) { d2min = od; jmin = oj; }
    }
    if (!active || sub != 0) return;
    double v = num / den;
    const double dmin = __dsqrt_rn(d2min);
    if (dmin < zero_eps) {
        // nearest by d (not d^2): lowest j among perspectives whose rounded d equals dmin
        int jbest = jmin;
        for (int j = 0; j < jmin; ++j) {
            const double d2 = dist2(x0, x1, x2, P[3 * (size_t)j], P[3 * (size_t)j + 1], P[3 * (size_t)j + 2]);
            if (__dsqrt_rn(d2) == dmin) { jbest = j; break; }
        }
        v = G[jbest];
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

}  // namespace

nbt_status launch_idbuf_push(nbt_ctx ctx, nbt_idbuf_s *b, const double *d_xyz, const double *d_gain, int32_t n)
{
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
    if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_q * 8))) return st;
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    dim3 grid((n_q + kQueries - 1) / kQueries, b->capacity);
    k_idw_entry<<<grid, kThreads, 0, ctx->stream>>>(b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, a.pos,
                                                     n_q, power_p, zero_eps, ctx->idw_tmp.as<double>());
    NBT_LAUNCHED(ctx);
    k_info_cost<<<(a.n_traj + 63) / 64, 64, 0, ctx->stream>>>(ctx->idw_tmp.as<double>(), b->d_meta, b->capacity, a,
                                                              normalize, ctx->d_err);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_idw(nbt_ctx ctx, const nbt_idbuf_s *b, const double *d_q, int32_t n_q, double power_p,
                      double zero_eps, int32_t normalize, double *d_out)
{
    if (n_q == 0) return NBT_OK;
    nbt_status st;
    if ((st = ctx->idw_tmp.ensure((size_t)b->capacity * n_q * 8))) return st;
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    dim3 grid((n_q + kQueries - 1) / kQueries, b->capacity);
    k_idw_entry<<<grid, kThreads, 0, ctx->stream>>>(b->d_xyz, b->d_gain, b->max_persp, b->d_meta, b->capacity, d_q,
                                                     n_q, power_p, zero_eps, ctx->idw_tmp.as<double>());
    NBT_LAUNCHED(ctx);
    k_idw_combine<<<(n_q + 127) / 128, 128, 0, ctx->stream>>>(ctx->idw_tmp.as<double>(), b->d_meta, b->capacity,
                                                               n_q, normalize, d_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
