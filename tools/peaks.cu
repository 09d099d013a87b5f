// Measured peaks of the resources that bound the ID walk (VERDICT r01
// item 3): integer issue on the ALU pipe (LOP3, IADD3, SHF, ISETP, PRMT) and on the FMA pipe
// (IMAD, with three register sources and with an immediate), their 1:1 mix, the FP32 FMA pipe
// for comparison, and the read bandwidth of the L2 (buffer resident in L2, loads that bypass
// L1) and of L1 (buffer per block resident in L1).
//
// Every throughput kernel runs 8 independent dependency chains per thread in an unrolled
// loop of inline-PTX instructions (cuobjdump -sass build/peaks shows the opcodes), on
// every SM with 32 resident warps.  The SM clock during each run is measured on the device
// (clock64 vs %globaltimer), so lanes/clk/SM does not depend on the clock assumption.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/peaks.cu -o build/peaks
//   ./build/peaks > profiles/r02_peaks.json
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ __forceinline__ uint64_t gtimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

enum Op {
    kLop3_3r,   // LOP3.LUT d, a, b, c          (ALU pipe, 3 register sources)
    kIadd_2r,   // two-input integer add (2 register sources)
    kIadd3,     // IADD3 d, a, b, c            (ALU pipe)
    kShf,       // SHF.R.U32.HI d, a, imm      (ALU pipe, 1 register source)
    kImad_3r,   // IMAD d, a, b, c             (FMA pipe, 3 register sources)
    kImad_imm,  // IMAD d, a, imm, c           (FMA pipe, 2 register sources)
    kMix,       // LOP3 (3r) and IMAD (3r) alternating, 1:1
    kMixImm,    // LOP3 (2r, another chain) and IMAD (imm) alternating, 1:1
    kFfma_3r,   // FFMA d, a, b, c
    kFfma_imm,  // FFMA d, a, imm, c
    kDfma,      // DFMA d, a, b, c           (FP64 pipe; the IDW's arithmetic)
    kNumOps
};
const char *kOpName[kNumOps] = {"lop3_3reg", "iadd_2reg", "iadd3_3reg", "shf_1reg", "imad_3reg", "imad_imm",
                                "mix_lop3_imad_3reg", "mix_lop3_imad_imm", "ffma_3reg", "ffma_imm", "dfma"};
const char *kOpPipe[kNumOps] = {"alu", "alu", "alu", "alu", "fma", "fma", "alu+fma", "alu+fma", "fma", "fma", "fp64"};

constexpr int kChains = 8;
constexpr int kUnroll = 16;     // instructions per chain per loop iteration

template <int OP>
__device__ __forceinline__ void step(uint32_t (&x)[kChains], uint32_t a, uint32_t b, int u)
{
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        if (OP == kLop3_3r) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if (OP == kIadd_2r) {
            asm volatile("add.s32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
        } else if (OP == kIadd3) {
            asm volatile("add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if (OP == kShf) {
            asm volatile("shf.l.wrap.b32 %0, %0, %0, 3;" : "+r"(x[c]));
        } else if (OP == kImad_3r) {
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if (OP == kImad_imm) {
            asm volatile("mad.lo.u32 %0, %0, 1664525, %1;" : "+r"(x[c]) : "r"(b));
        } else if (OP == kMix) {
            if (u & 1)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            else
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if (OP == kMixImm) {
            if (u & 1)
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(x[c]) : "r"(x[(c + 1) % kChains]));
            else
                asm volatile("mad.lo.u32 %0, %0, 1664525, %1;" : "+r"(x[c]) : "r"(b));
        } else if (OP == kFfma_3r) {
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        } else if (OP == kFfma_imm) {
            asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFE, %1;" : "+r"(x[c]) : "r"(b));
        }
    }
}

// SASS instructions each step() issues per chain: ptxas fuses two dependent adds into one
// three-input IADD3 (checked with cuobjdump -sass), so the kIadd_2r chain issues one IADD3
// per two PTX adds and the kIadd3 form one per step.
constexpr double instrs_per_step(int op) { return op == kIadd_2r ? 0.5 : 1.0; }

// DFMA chains on doubles (the FP64 pipe)
__global__ void __launch_bounds__(256) k_issue_f64(int iters, uint32_t seed, uint32_t *sink, unsigned long long *clk)
{
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
    const double m = 0.999999 + 1e-9 * (seed + threadIdx.x), d = 1e-7 * (threadIdx.x + 1);
    const uint64_t c0 = clock64(), t0 = gtimer();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
            for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(m), "d"(d));
    }
    const uint64_t c1 = clock64(), t1 = gtimer();
    double acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc += x[c];
    if (acc == 12345.0) sink[threadIdx.x] = 1;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = c1 - c0;
        clk[1] = t1 - t0;
    }
}

template <int OP>
__global__ void __launch_bounds__(256) k_issue(int iters, uint32_t seed, uint32_t *sink, unsigned long long *clk)
{
    uint32_t x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B9u;
    // per-thread operands, so ptxas keeps them in vector (not uniform) registers
    const uint32_t a = (seed * threadIdx.x) | 1u, b = (seed + threadIdx.x) ^ 0x5bd1e995u;
    const uint64_t c0 = clock64(), t0 = gtimer();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) step<OP>(x, a, b, u);
    }
    const uint64_t c1 = clock64(), t1 = gtimer();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= x[c];
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;     // keeps the chains alive
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = c1 - c0;
        clk[1] = t1 - t0;
    }
}

// L2 read bandwidth: every warp reads 16-byte vectors with ld.global.cg (cached in L2 only),
// grid-stride over a buffer that stays resident in L2.
__global__ void __launch_bounds__(512) k_l2_read(const uint4 *__restrict__ buf, size_t n16, int passes, uint32_t *sink)
{
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(buf + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

// L1 hit bandwidth: each block re-reads its own 32 KB slice with ld.global.ca (4-byte loads,
// 32 distinct consecutive words per warp request = one 128-B line) -- the request shape of a
// coherent walk -- and, in the scattered form, 32 distinct lines per request (each lane its
// own 128-B line), the shape of an incoherent one.
template <bool SCATTER>
__global__ void __launch_bounds__(256) k_l1_read(const uint32_t *__restrict__ buf, int iters, uint32_t *sink)
{
    const uint32_t *slice = buf + (size_t)blockIdx.x * 8192;   // 32 KB per block
    uint32_t acc = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int line = (warp * 16 + u + it) & 255;       // 256 lines of 128 B
            const int w = SCATTER ? (((line + lane * 8) & 255) * 32 + (lane & 31)) : (line * 32 + lane);
            uint32_t v;
            asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(slice + w));
            acc += v;
        }
    }
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
}

struct Res {
    double lanes_per_clk_sm, ops_per_s, mhz;
};

template <int OP>
Res run_issue(int sms, int iters)
{
    uint32_t *sink;
    unsigned long long *clk;
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMalloc(&clk, 16));
    const int blocks = sms * 8;          // 8 x 256 threads = 64 warps per SM
    auto launch = [&](int it) {
        if (OP == kDfma) k_issue_f64<<<blocks, 256>>>(it, 7u, sink, clk);
        else k_issue<OP><<<blocks, 256>>>(it, 7u, sink, clk);
    };
    launch(iters / 8);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best = 0, mhz = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        launch(iters);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long h[2];
        CK(cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost));
        const double ops = (double)blocks * 256 * iters * kUnroll * kChains * instrs_per_step(OP);
        const double r = ops / (ms * 1e-3);
        if (r > best) {
            best = r;
            mhz = h[1] ? (double)h[0] / (double)h[1] * 1e3 : 0;
        }
    }
    CK(cudaFree(sink));
    CK(cudaFree(clk));
    return Res{best / ((double)sms * mhz * 1e6), best, mhz};
}

double run_l2(size_t bytes, int sms)
{
    uint4 *buf;
    uint32_t *sink;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMemset(buf, 1, bytes));
    const size_t n16 = bytes / 16;
    const int blocks = sms * 4;
    k_l2_read<<<blocks, 512>>>(buf, n16, 2, sink);      // warm: the buffer becomes L2-resident
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best = 0;
    const int passes = 20;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        k_l2_read<<<blocks, 512>>>(buf, n16, passes, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::max(best, (double)bytes * passes / (ms * 1e-3) / 1e9);
    }
    CK(cudaFree(buf));
    CK(cudaFree(sink));
    return best;
}

template <bool SCATTER>
double run_l1(int sms, double *requests_per_clk_sm, double mhz)
{
    uint32_t *buf, *sink;
    const int blocks = sms * 4;
    CK(cudaMalloc(&buf, (size_t)blocks * 32768));
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMemset(buf, 1, (size_t)blocks * 32768));
    const int iters = 4000;
    k_l1_read<SCATTER><<<blocks, 256>>>(buf, 100, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        k_l1_read<SCATTER><<<blocks, 256>>>(buf, iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double req = (double)blocks * 8 * iters * 16;      // warp-level load requests
        best = std::max(best, req / (ms * 1e-3));
    }
    *requests_per_clk_sm = best / (sms * mhz * 1e6);
    CK(cudaFree(buf));
    CK(cudaFree(sink));
    return best * 128.0 / 1e9;          // GB/s of requested bytes (32 lanes x 4 B)
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int iters = 2000;
    Res r[kNumOps] = {run_issue<kLop3_3r>(sms, iters),  run_issue<kIadd_2r>(sms, iters),
                      run_issue<kIadd3>(sms, iters),    run_issue<kShf>(sms, iters),
                      run_issue<kImad_3r>(sms, iters),  run_issue<kImad_imm>(sms, iters),
                      run_issue<kMix>(sms, iters),      run_issue<kMixImm>(sms, iters),
                      run_issue<kFfma_3r>(sms, iters),  run_issue<kFfma_imm>(sms, iters),
                      run_issue<kDfma>(sms, iters)};
    double mhz = 0;
    for (auto &x : r) mhz = std::max(mhz, x.mhz);
    double best_int = 0;
    for (int k = 0; k < kNumOps; ++k)
        if (k != kFfma_3r && k != kFfma_imm && k != kDfma) best_int = std::max(best_int, r[k].ops_per_s);
    const double l2_32 = run_l2(32ull << 20, sms), l2_64 = run_l2(64ull << 20, sms);
    double l1_req_c = 0, l1_req_s = 0;
    const double l1_c = run_l1<false>(sms, &l1_req_c, mhz), l1_s = run_l1<true>(sms, &l1_req_s, mhz);
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"sm_mhz_measured\": %.1f,\n", prop.name, sms, mhz);
    printf("  \"how\": \"tools/peaks.cu: 148 SMs x 8 blocks x 256 threads, 8 independent chains per thread of "
           "inline-PTX instructions, best of 3 (CUDA events); SM clock from clock64 vs globaltimer during the run\",\n");
    printf("  \"issue\": {\n");
    for (int k = 0; k < kNumOps; ++k)
        printf("    \"%s\": {\"pipe\": \"%s\", \"warp_instr_per_clk_per_smsp\": %.3f, \"lanes_per_clk_per_sm\": %.1f, "
               "\"ops_per_s\": %.4e}%s\n",
               kOpName[k], kOpPipe[k], r[k].lanes_per_clk_sm / 128.0, r[k].lanes_per_clk_sm, r[k].ops_per_s,
               k + 1 < kNumOps ? "," : "");
    printf("  },\n");
    printf("  \"int32_peak_ops_per_s\": %.4e,\n", best_int);
    printf("  \"int32_peak_tops\": %.3f,\n", best_int / 1e12);
    printf("  \"int32_peak_lanes_per_clk_per_sm\": %.1f,\n", best_int / (sms * mhz * 1e6));
    printf("  \"l2_read_gbs\": {\"32MiB\": %.1f, \"64MiB\": %.1f},\n", l2_32, l2_64);
    printf("  \"l2_read_peak_gbs\": %.1f,\n", std::max(l2_32, l2_64));
    printf("  \"l1_read\": {\"coherent_gbs\": %.1f, \"coherent_warp_requests_per_clk_per_sm\": %.3f, "
           "\"scattered_gbs\": %.1f, \"scattered_warp_requests_per_clk_per_sm\": %.3f}\n",
           l1_c, l1_req_c, l1_s, l1_req_s);
    printf("}\n");
    return 0;
}
