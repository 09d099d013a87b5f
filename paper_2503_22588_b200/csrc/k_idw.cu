// IDW query over the ID ring buffer (Eq. 4).
//
//   G(x) = sum_u w_u * [ sum_j g_P,j d_j(x)^-p / sum_j d_j(x)^-p ]
//
// over the buffered clouds u = oldest..newest with w_u = 1/(m-u) (newest weighs 1,
// reading Q21), each cloud's own perspectives (Q20) and all of them (Q22); if the
// nearest perspective is closer than zero_eps the bracket is its gain (Q23).
// One warp per query: lanes stride over an entry's perspectives, FP64 throughout
// (p = 2 needs no pow: d^-2 = 1/d^2), warp shuffles combine the partial sums and the
// (distance, index) argmin -- the nearest-perspective decision is made on
// correctly-rounded d = sqrt(d^2) so it is exactly reproducible.
#include "nbt_internal.cuh"

namespace nbt {
namespace {

constexpr int kWarps = 8;

__global__ void __launch_bounds__(kWarps * 32)
    k_idw_query(const double *__restrict__ xyz, const double *__restrict__ gain, int32_t max_persp, IdwEntries E,
                const double *__restrict__ q, int32_t n_q, double power_p, double zero_eps, int32_t normalize,
                double *__restrict__ out)
{
    const int lane = threadIdx.x & 31;
    const int qi = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (qi >= n_q) return;
    const double x0 = q[3 * (size_t)qi], x1 = q[3 * (size_t)qi + 1], x2 = q[3 * (size_t)qi + 2];
    const bool p2 = power_p == 2.0;
    const double hp = -0.5 * power_p;
    double G = 0.0, wsum = 0.0;
    for (int e = 0; e < E.m; ++e) {
        const double *P = xyz + (size_t)E.slot[e] * max_persp * 3;
        const double *Gn = gain + (size_t)E.slot[e] * max_persp;
        const int np = E.size[e];
        double num = 0.0, den = 0.0, dmin = __longlong_as_double(0x7ff0000000000000LL);
        int jmin = 0x7fffffff;
        for (int j = lane; j < np; j += 32) {
            double dx = __dsub_rn(x0, P[3 * j]), dy = __dsub_rn(x1, P[3 * j + 1]), dz = __dsub_rn(x2, P[3 * j + 2]);
            double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            double d = __dsqrt_rn(d2);
            if (d < dmin) { dmin = d; jmin = j; }
            double w = p2 ? __drcp_rn(d2) : pow(d2, hp);
            num = fma(Gn[j], w, num);
            den += w;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, off);
            den += __shfl_xor_sync(0xffffffffu, den, off);
            double od = __shfl_xor_sync(0xffffffffu, dmin, off);
            int oj = __shfl_xor_sync(0xffffffffu, jmin, off);
            if (od < dmin || (od == dmin && oj < jmin)) { dmin = od; jmin = oj; }
        }
        double v = (dmin < zero_eps) ? Gn[jmin] : num / den;
        double wu = 1.0 / (double)(E.m - e);
        G += wu * v;
        wsum += wu;
    }
    if (lane == 0) out[qi] = normalize ? G / wsum : G;
}

}  // namespace

nbt_status launch_idw(nbt_ctx ctx, const nbt_idbuf_s *b, const IdwEntries &E, const double *d_q, int32_t n_q,
                      double power_p, double zero_eps, int32_t normalize, double *d_out)
{
    if (n_q == 0) return NBT_OK;
    ProfScope ps(ctx, NBT_KERNEL_IDW);
    k_idw_query<<<(n_q + kWarps - 1) / kWarps, kWarps * 32, 0, ctx->stream>>>(
        b->d_xyz, b->d_gain, b->max_persp, E, d_q, n_q, power_p, zero_eps, normalize, d_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
