// Instruction-mix ceiling of the ID walk: the exact DDA step of
// dda.cuh (walk_step, int32 decision terms, linear layout) run on registers only -- no map
// loads, no rays to set up, every lane busy -- and the same step plus the per-visit code
// extraction of k_id_trace (rotate + pack of a register word).  The visits/s it reaches is
// what the kernel's instruction mix alone allows on this GPU; bench.py's in-grid lookups/s
// divided by it says how much the loads, the ray set-up, idle lanes and speculation cost.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        -I paper_2503_22588_b200/csrc tools/dda_step_peak.cu -o build/dda_step_peak
//   ./build/dda_step_peak
#include <cstdio>
#include <cstdlib>

#include "dda.cuh"

using namespace nbt;
using namespace nbt::dda;

constexpr int kSteps = 16;          // one speculative batch of k_id_trace

template <bool EXTRACT>
__global__ void __launch_bounds__(256) k_step_peak(int iters, uint32_t seed, uint32_t *sink)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    // a ray with slopes of similar size on the three axes (every axis steps)
    Walk<int> w{};
    const int o[3] = {(int)(100 << 12) + (int)(t & 4095), (int)(120 << 12) + (int)((t * 7) & 4095),
                      (int)(90 << 12) + (int)((t * 13) & 4095)};
    const int e[3] = {o[0] + (int)(600 << 12) + (int)(seed & 1023), o[1] + (int)(500 << 12),
                      o[2] - (int)(550 << 12)};
    walk_setup(w, o, e);
    w.dX = 1; w.dY = 320; w.ndZ = 320 * 320;
    w.idx = t;
    MapView m{};
    uint32_t acc = 0, word = seed ^ t;
    for (int it = 0; it < iters; ++it) {
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < kSteps; ++k) {
            if (EXTRACT) {
                const uint32_t rot = (w.idx << 1) - 2 * k;
                bits |= __funnelshift_r(word, word, rot) & (3u << (2 * k));
            }
            walk_step<int, kLayoutLinear, false>(w, m);
        }
        acc += EXTRACT ? __popc(bits & 0x55555555u) : w.idx;
        word = word * 1664525u + 1013904223u;
    }
    if (acc == 0x12345678u) sink[t] = acc + w.qxy + w.qxz + w.qyz;   // never true; keeps the work
}

template <bool EXTRACT>
double run(int sms, int iters)
{
    uint32_t *sink;
    cudaMalloc(&sink, sizeof(uint32_t) * 256 * 64 * 1024);
    const int blocks = sms * 8;
    k_step_peak<EXTRACT><<<blocks, 256>>>(iters / 10, 1u, sink);      // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_step_peak<EXTRACT><<<blocks, 256>>>(iters, 1u, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(sink);
    const double steps = (double)blocks * 256 * iters * kSteps;
    return steps / (ms * 1e-3);
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int iters = 4000;
    const double s0 = run<false>(sms, iters), s1 = run<true>(sms, iters);
    const double peak = (double)sms * 128 * 1.965e9;          // int32 lanes x max clock
    printf("{\"sms\": %d, \"dda_step_only_per_s\": %.4e, \"dda_step_plus_extract_per_s\": %.4e, "
           "\"alg_int32_ops_per_s_at_extract\": %.4e, \"frac_of_alu_peak\": %.3f}\n",
           sms, s0, s1, 13.0 * s1, 13.0 * s1 / peak);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
