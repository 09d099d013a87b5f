// Instruction-mix ceiling of the ID walk: the exact DDA step of
// dda.cuh (walk_step, int32 decision terms, linear layout) run on registers only -- no map
// loads, no rays to set up, every lane busy -- and the same step plus the per-visit code
// packing of k_id_trace: MODE 1 = the 2-bit store's (rotate of a register word by the code's
// bit offset + funnel shift into the batch word), MODE 2 = the byte stores' (shift-add of a
// register byte).  The visits/s it reaches is
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

template <int MODE>
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
    w.dX = 2; w.dY = 640; w.ndZ = 640 * 320;       // the 2-bit store's bit-offset steps
    w.idx = t;
    MapView m{};
    uint32_t acc = 0, word = seed ^ t;
    for (int it = 0; it < iters; ++it) {
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < kSteps; ++k) {
            if (MODE == 1) bits = __funnelshift_l(__funnelshift_l(word, word, w.idx), bits, 2);
            if (MODE == 2) bits = bits * 4u + ((word >> (w.idx & 24)) & 3u);
            walk_step<int, kLayoutLinear, false>(w, m);
        }
        acc += MODE ? __popc(bits & 0x55555555u) : w.idx;
        word = word * 1664525u + 1013904223u;
    }
    if (acc == 0x12345678u) sink[t] = acc + w.qxy + w.qxz + w.qyz;   // never true; keeps the work
}

template <int MODE>
double run(int sms, int iters)
{
    uint32_t *sink;
    cudaMalloc(&sink, sizeof(uint32_t) * 256 * 64 * 1024);
    const int blocks = sms * 8;
    k_step_peak<MODE><<<blocks, 256>>>(iters / 10, 1u, sink);      // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_step_peak<MODE><<<blocks, 256>>>(iters, 1u, sink);
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
    const double s0 = run<0>(sms, iters), s1 = run<1>(sms, iters), s2 = run<2>(sms, iters);
    const double peak = 35.914e12;     // measured best integer mix (profiles/r02_peaks.json), 12 ops per visit
    printf("{\"sms\": %d, \"dda_step_only_per_s\": %.4e, \"step_plus_pack_2bit_per_s\": %.4e, "
           "\"step_plus_pack_byte_per_s\": %.4e, \"frac_of_int32_peak_2bit\": %.3f, \"frac_of_int32_peak_byte\": %.3f}\n",
           sms, s0, s1, s2, 12.0 * s1 / peak, 12.0 * s2 / peak);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
