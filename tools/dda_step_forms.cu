// Instruction-form probe of the exact DDA step: the same int32 step as
// dda.cuh's walk_step, written three ways, run on registers only (every lane busy, the 2-bit
// store's per-visit rotate + funnel-shift packing, no map loads) so that only the step's
// instruction count and operand shape differ.
//   FORM 0: the round-1/2 hot path (0/1 flags from the sign bits, 9 multiply-adds by the flags)
//   FORM 1: predicates (3 setp + 1 or.pred) and 9 predicated adds, written in PTX (dda.cuh's
//           walk_step since session 4 of round 2; FORM 3 calls it)
//   FORM 2: the same predicates, the updates as C++ conditionals (ptxas picks the forms)
// All forms must end on the same decision terms and index (checksum printed per form).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        -I paper_2503_22588_b200/csrc tools/dda_step_forms.cu -o build/dda_step_forms
#include <cstdio>
#include <cstdlib>

#include "dda.cuh"

using namespace nbt;
using namespace nbt::dda;

constexpr int kSteps = 16;

template <int FORM>
__device__ __forceinline__ void step(Walk<int> &w, const MapView &m)
{
    if constexpr (FORM == 0) {
        const int t1 = w.qxy & w.qxz;
        const int t2 = w.qyz & ~t1;
        const int px = (int)((unsigned)t1 >> 31);
        const int py = (int)((unsigned)t2 >> 31);
        const int npz = px + py - 1;
        w.qxy = mad_i32(px, w.ay, mad_i32(py, w.nax, w.qxy));
        w.qxz = mad_i32(px, w.az, mad_i32(npz, w.ax, w.qxz));
        w.qyz = mad_i32(py, w.az, mad_i32(npz, w.ay, w.qyz));
        w.idx = (uint32_t)mad_i32(px, w.dX, mad_i32(py, w.dY, mad_i32(npz, w.ndZ, (int)w.idx)));
    } else if constexpr (FORM == 3) {
        walk_step<int, kLayoutLinear, false>(w, m);
    } else if constexpr (FORM == 1) {
        asm("{\n\t.reg .pred t, px, py, pxy;\n\t"
            "setp.lt.s32 t, %1, 0;\n\t"
            "setp.lt.and.s32 px, %0, 0, t;\n\t"
            "setp.lt.and.s32 py, %2, 0, !px;\n\t"
            "or.pred pxy, px, py;\n\t"
            "@px add.s32 %0, %0, %4;\n\t"
            "@px add.s32 %1, %1, %5;\n\t"
            "@px add.s32 %3, %3, %7;\n\t"
            "@py sub.s32 %0, %0, %6;\n\t"
            "@py add.s32 %2, %2, %5;\n\t"
            "@py add.s32 %3, %3, %8;\n\t"
            "@!pxy sub.s32 %1, %1, %6;\n\t"
            "@!pxy sub.s32 %2, %2, %4;\n\t"
            "@!pxy sub.s32 %3, %3, %9;\n\t}"
            : "+r"(w.qxy), "+r"(w.qxz), "+r"(w.qyz), "+r"(w.idx)
            : "r"(w.ay), "r"(w.az), "r"(w.ax), "r"(w.dX), "r"(w.dY), "r"(w.ndZ));
    } else {
        const bool px = (w.qxy < 0) & (w.qxz < 0);
        const bool py = !px & (w.qyz < 0);
        const bool pz = !(px | py);
        if (px) { w.qxy += w.ay; w.qxz += w.az; w.idx += w.dX; }
        if (py) { w.qxy -= w.ax; w.qyz += w.az; w.idx += w.dY; }
        if (pz) { w.qxz -= w.ax; w.qyz -= w.ay; w.idx -= w.ndZ; }
    }
}

template <int FORM>
__global__ void __launch_bounds__(256) k_forms(int iters, uint32_t seed, uint32_t *sink)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    Walk<int> w{};
    const int o[3] = {(int)(100 << 12) + (int)(t & 4095), (int)(120 << 12) + (int)((t * 7) & 4095),
                      (int)(90 << 12) + (int)((t * 13) & 4095)};
    const int e[3] = {o[0] + (int)(600 << 12) + (int)(seed & 1023), o[1] + (int)(500 << 12),
                      o[2] - (int)(550 << 12)};
    walk_setup(w, o, e);
    w.dX = 2; w.dY = 640; w.ndZ = 640 * 320;
    w.idx = t;
    MapView m{};
    uint32_t acc = 0, word = seed ^ t;
    for (int it = 0; it < iters; ++it) {
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < kSteps; ++k) {
            bits = __funnelshift_l(__funnelshift_l(word, word, w.idx), bits, 2);
            step<FORM>(w, m);
        }
        acc += __popc(bits & 0x55555555u);
        word = word * 1664525u + 1013904223u;
        // keep the terms bounded: the probe ray is periodic in the lattice
        if ((it & 255) == 255) { walk_setup(w, o, e); w.dX = 2; w.dY = 640; w.ndZ = 640 * 320; w.idx = t + it; }
    }
    sink[t] = acc + w.qxy + w.qxz + w.qyz + w.idx;
}

template <int FORM>
void run(int sms, int iters, uint32_t *sink)
{
    const int blocks = sms * 8;
    k_forms<FORM><<<blocks, 256>>>(iters / 10, 1u, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        k_forms<FORM><<<blocks, 256>>>(iters, 1u, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const int n = blocks * 256;
    uint32_t *h = (uint32_t *)malloc(sizeof(uint32_t) * n);
    cudaMemcpy(h, sink, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost);
    unsigned long long cs = 0;
    for (int i = 0; i < n; ++i) cs = cs * 1000003ull + h[i];
    free(h);
    const double steps = (double)n * iters * kSteps;
    printf("{\"form\": %d, \"visits_per_s\": %.4e, \"ms\": %.3f, \"checksum\": \"%016llx\"}\n", FORM,
           steps / (best * 1e-3), best, cs);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *sink;
    cudaMalloc(&sink, sizeof(uint32_t) * sms * 8 * 256);
    const int iters = 4000;
    run<0>(sms, iters, sink);
    run<1>(sms, iters, sink);
    run<2>(sms, iters, sink);
    run<3>(sms, iters, sink);
    run<0>(sms, iters, sink);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
