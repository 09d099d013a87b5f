// Perspective sampling by Eq. 1.
//
// p_P = p_POI + r_S * X_R^(1/3) * X / ||X||  with X ~ N(0, I_3) (Muller's method,
// P:145) and X_R ~ U(0,1) (reading Q1; the printed "G(0,1)" is garbled), or X_R = 1
// in surface mode (Q3).  Draws come from a counter-based Philox4x32-10 generator so
// that every perspective j is independent of the launch shape (reading Q29):
// counter (j, attempt, 0, 0) -> four uniforms for two Box-Muller pairs,
// counter (j, attempt, 1, 0) -> X_R.  ||X|| < 1e-12 is resampled.
#include "nbt_internal.cuh"

namespace nbt {
namespace {

struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox10(U4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ double unit_open(uint32_t b) { return ((double)b + 0.5) * 2.3283064365386963e-10; }

__global__ void k_sample_perspectives(double px, double py, double pz, double r_s, int32_t n, uint32_t k0,
                                      uint32_t k1, int32_t mode, double *__restrict__ out)
{
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double two_pi = 6.283185307179586;
    for (uint32_t attempt = 0;; ++attempt) {
        U4 b = philox10(U4{(uint32_t)j, attempt, 0u, 0u}, k0, k1);
        double u0 = unit_open(b.x), u1 = unit_open(b.y), u2 = unit_open(b.z), u3 = unit_open(b.w);
        double r01 = sqrt(-2.0 * log(u0)), r23 = sqrt(-2.0 * log(u2));
        double s1, c1, s3, c3;
        sincos(two_pi * u1, &s1, &c1);
        sincos(two_pi * u3, &s3, &c3);
        double X0 = r01 * c1, X1 = r01 * s1, X2 = r23 * c3;
        double nx = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(X0, X0), __dmul_rn(X1, X1)), __dmul_rn(X2, X2)));
        if (nx < 1e-12) continue;
        double xr = 1.0;
        if (mode == NBT_SAMPLE_BALL) xr = unit_open(philox10(U4{(uint32_t)j, attempt, 1u, 0u}, k0, k1).x);
        double scale = r_s * cbrt(xr);
        out[3 * (size_t)j + 0] = px + scale * (X0 / nx);
        out[3 * (size_t)j + 1] = py + scale * (X1 / nx);
        out[3 * (size_t)j + 2] = pz + scale * (X2 / nx);
        return;
    }
}

}  // namespace

nbt_status launch_sample(nbt_ctx ctx, const double poi[3], double r_s, int32_t n, uint64_t seed, int32_t mode,
                         double *d_out)
{
    if (n == 0) return NBT_OK;
    ProfScope ps(ctx, NBT_KERNEL_SAMPLE);
    k_sample_perspectives<<<(n + 127) / 128, 128, 0, ctx->stream>>>(poi[0], poi[1], poi[2], r_s, n,
                                                                     (uint32_t)seed, (uint32_t)(seed >> 32), mode,
                                                                     d_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
