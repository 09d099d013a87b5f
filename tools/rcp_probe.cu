// Accuracy of rcp.approx.ftz.f64 (MUFU.RCP64H) alone and after one / two Newton steps, over
// 2^24 random doubles in [1e-6, 1e3) (the IDW's d^2 range): max relative error vs the IEEE
// reciprocal.  Decides how many Newton steps k_idw_entry needs for its 1e-12 tolerance.
#include <cstdio>
#include <cstdint>
#include <cmath>
__global__ void k(double *out)
{
    double m0 = 0, m1 = 0, m2 = 0;
    uint64_t s = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    for (int i = 0; i < 256; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        const double u = (double)(s >> 11) * 0x1.0p-53;
        const double x = exp(log(1e-6) + u * (log(1e3) - log(1e-6)));
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        const double ex = __drcp_rn(x);
        m0 = fmax(m0, fabs(r - ex) / ex);
        double e = fma(-x, r, 1.0);
        double r1 = fma(r, e, r);
        m1 = fmax(m1, fabs(r1 - ex) / ex);
        e = fma(-x, r1, 1.0);
        double r2 = fma(r1, e, r1);
        m2 = fmax(m2, fabs(r2 - ex) / ex);
    }
    out[3 * (blockIdx.x * blockDim.x + threadIdx.x) + 0] = m0;
    out[3 * (blockIdx.x * blockDim.x + threadIdx.x) + 1] = m1;
    out[3 * (blockIdx.x * blockDim.x + threadIdx.x) + 2] = m2;
}
int main()
{
    const int n = 65536;
    double *d, *h = new double[3 * n];
    cudaMalloc(&d, 3 * n * sizeof(double));
    k<<<n / 256, 256>>>(d);
    cudaMemcpy(h, d, 3 * n * sizeof(double), cudaMemcpyDeviceToHost);
    double m[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < 3; ++j) m[j] = fmax(m[j], h[3 * i + j]);
    printf("{\"samples\": %d, \"rcp_approx_max_rel\": %.3e, \"one_newton_max_rel\": %.3e, \"two_newton_max_rel\": %.3e}\n",
           n * 256, m[0], m[1], m[2]);
    return 0;
}
