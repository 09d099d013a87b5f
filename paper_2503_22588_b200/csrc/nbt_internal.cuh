// Internal declarations shared by the libnbt translation units (product code only;
// nothing here is visible across the C ABI).  Citations: P:n = PAPER.md line n.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "nbt.h"

namespace nbt {

// ----------------------------------------------------------------- errors

void set_error(const std::string &msg);
nbt_status fail(nbt_status s, const std::string &msg);
nbt_status cuda_fail(cudaError_t e, const char *what);

#define NBT_CUDA(call)                                                   \
    do {                                                                 \
        cudaError_t e_ = (call);                                         \
        if (e_ != cudaSuccess) return ::nbt::cuda_fail(e_, #call);       \
    } while (0)

#define NBT_LAUNCHED(ctx)                                                \
    do {                                                                 \
        (ctx)->launches++;                                               \
        cudaError_t e_ = cudaGetLastError();                             \
        if (e_ != cudaSuccess) return ::nbt::cuda_fail(e_, "kernel launch"); \
    } while (0)

// Thickness of the sentinel shell around the stored grid (k_map.cu); bounds the
// walk's speculative look-ahead (k_id.cu: batch size, twice that when pipelined).
#ifndef NBT_BORDER
#define NBT_BORDER 16
#endif
constexpr int kBorder = NBT_BORDER;

// Map store layouts (k_map.cu).  Linear: x-fastest rows inside a kBorder sentinel shell.
// Morton: the voxel index interleaves the coordinate bits (x0 y0 z0 x1 y1 z1 ...) inside a
// cube of side P = 2^pbits >= max(n) + 2 kBorder, so one 128-byte line holds an 8x8x8
// block and one 32-byte sector a 4x4x8 block; coordinates wrap modulo P, and every
// voxel of the cube outside the grid holds the sentinel.
enum : int { kLayoutLinear = 0, kLayoutMorton = 1 };

// Spread the low 10 bits of v to bit positions 0, 3, 6, ..., 27.
__host__ __device__ __forceinline__ uint32_t dilate3(uint32_t v)
{
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

// Inverse of dilate3 on bit positions 0, 3, 6, ...
__host__ __device__ __forceinline__ uint32_t compact3(uint32_t v)
{
    v &= 0x09249249u;
    v = (v ^ (v >> 2)) & 0x030C30C3u;
    v = (v ^ (v >> 4)) & 0x0300F00Fu;
    v = (v ^ (v >> 8)) & 0x030000FFu;
    v = (v ^ (v >> 16)) & 0x3ffu;
    return v;
}

// ----------------------------------------------------------- buffers

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    nbt_status ensure(size_t bytes);
    void release();
    template <class T> T *as() const { return static_cast<T *>(p); }
};

// Pinned host staging area, reused after its last async copy completed.
struct HostStage {
    void *p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
    nbt_status acquire(size_t bytes);   // waits for the previous copy out of / into it
    nbt_status mark(cudaStream_t s);    // record the copy just enqueued
    void release();
};

// True while the calling thread's ctx stream is being captured into a CUDA graph:
// buffers must not grow (warm up first) and nothing may synchronize.
extern thread_local bool g_capturing;

struct CapPair {
    int kernel;
    cudaEvent_t start, end;
};

// Per-kernel-family event timing (nbt_ctx_set_profiling).
struct Profiler {
    bool on = false;
    uint32_t mask = ~0u;              // kernel families recorded (bit = NBT_KERNEL_*)
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[NBT_KERNEL_COUNT];
    double ms[NBT_KERNEL_COUNT] = {0};
    uint64_t n[NBT_KERNEL_COUNT] = {0};
    cudaEvent_t take();
};

// RAII: records a start event at construction and an end event at destruction when
// profiling is on.
struct ProfScope {
    nbt_ctx ctx;
    int kernel;
    cudaEvent_t start = nullptr;
    ProfScope(nbt_ctx c, int k);
    ~ProfScope();
};

}  // namespace nbt

// ----------------------------------------------------------------- handles

// Tuning options of a ctx (nbt_ctx_set_option; none changes a result).
struct NbtOptions {
    int refill_min = 32;              // NBT_OPT_TRACE_REFILL_MIN (32: a warp refills when all lanes are idle)
    int chunk_min = 64;               // NBT_OPT_TRACE_CHUNK_MIN
    int carveout = 25;                // NBT_OPT_TRACE_CARVEOUT
    int delta_sort = 0;               // NBT_OPT_DELTA_SORT
    int filter_sort = 0;              // NBT_OPT_FILTER_SORT
    int h2d_mode = 0;                 // NBT_OPT_H2D_MODE
    int copy_threads = 0;             // NBT_OPT_COPY_THREADS (default set at ctx creation)
    int walk_width = 0;               // NBT_OPT_WALK_WIDTH
    int verbose = 0;                  // NBT_OPT_VERBOSE
};

struct nbt_ctx_s {
    int refs = 1;                     // 1 for the ctx itself + 1 per live map / ID buffer / graph
    bool closed = false;              // nbt_ctx_destroy called
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t launches = 0;
    int *d_err = nullptr;             // device-side validation status (nbt_status value)
    int *h_err = nullptr;             // pinned mirror
    NbtOptions opt;
    int trace_blocks_per_sm = 0;      // cached occupancy of the trace kernel (0: recompute at the next launch)
    int trace_bps[24] = {0};          // ... per instance [lockstep][wide][morton][store kind]
    // scratch
    nbt::DevBuf persp;                // staged perspective origins (n x 3 f64)
    nbt::DevBuf frames;               // per-perspective Q16 frames
    nbt::DevBuf totals;               // per-perspective u64 totals (U, F, O, L)
    nbt::DevBuf counter;              // work counter(s)
    nbt::DevBuf out_tmp;              // device staging for host outputs
    nbt::DevBuf deltas;               // staged map deltas
    nbt::DevBuf keys, keys_alt, cub_tmp;
    nbt::DevBuf queries, qout, idw_tmp, poses;
    nbt::DevBuf idw_done;             // IDW per-query-block completion counters (k_idw.cu)
    size_t idw_done_zeroed = 0;       // ... counters known to be zero ...
    void *idw_done_at = nullptr;      // ... at this address
    nbt::DevBuf dbg;                  // debug entry points
    nbt::HostStage stage_in[3];
    nbt::HostStage stage_out;
    nbt::Profiler prof;
    bool capturing = false;
    uint64_t cap_launches0 = 0;
    std::vector<nbt::CapPair> cap_pairs;  // profiling events recorded inside the capture
};

struct nbt_graph_s {
    nbt_ctx ctx = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t kernels = 0;                 // kernel nodes per launch
    std::vector<nbt::CapPair> pairs;
};

struct nbt_map_s {
    nbt_ctx ctx = nullptr;
    nbt_map_desc desc{};
    int layout = nbt::kLayoutLinear;
    int vbits = 2;                    // 2: 2-bit codes; 8: one byte per voxel
    bool prob = false;                // byte store also holds the Eq. 2 gain (f1)
    int pbits = 0;                    // Morton: cube side 2^pbits
    uint32_t px = 0, py = 0, pz = 0;  // linear: padded extents (kBorder sentinel voxels each side)
    uint64_t nvox_pad = 0;
    size_t nwords = 0;
    uint32_t *d_words = nullptr;      // 2-bit codes, 16 voxels per 32-bit word
    uint32_t *d_win = nullptr;        // delta winner per voxel (k_map.cu), lazily allocated
};

struct nbt_idbuf_s {
    nbt_ctx ctx = nullptr;
    int32_t capacity = 0, max_persp = 0;
    int32_t count = 0;                // host mirror of min(pushes, capacity) (validation only)
    int32_t *d_meta = nullptr;        // device: [0] = pushes so far, [1 + slot] = entry sizes
    double *d_xyz = nullptr;          // capacity x max_persp x 3
    double *d_gain = nullptr;         // capacity x max_persp
};

// Peer-memory gather of the IG cloud (multi-GPU): every rank's finalize writes
// its rows straight into all ranks' row buffers (mapped with CUDA IPC; over NVLink/NVSwitch
// when the owner is another GPU), so the all-gather is fused into the finalize kernel.
constexpr int kMaxGatherRanks = 16;
struct GatherDst {
    int n = 0;                                      // destinations
    double *xyz[kMaxGatherRanks] = {};
    double *gain[kMaxGatherRanks] = {};
    unsigned long long *counts[kMaxGatherRanks] = {};
};

// Ray-shard counts added straight into every rank's totals (the all-reduce of the ray split
// fused into the trace's count flushes: remote atomics over NVLink/NVSwitch).
struct PeerTotals {
    int n = 0;
    unsigned long long *t[kMaxGatherRanks] = {};
};

struct nbt_gather_s {
    nbt_ctx ctx = nullptr;
    int32_t rows = 0, world = 0, rank = 0;
    char *base = nullptr;             // local rows: xyz rows*24 | gain rows*8 | counts rows*32
    char *peer[kMaxGatherRanks] = {}; // rank r's rows (own: base; others: opened IPC mappings)
    PeerTotals *d_pt = nullptr;       // device copy of the peer-totals table (rewritten by every attach)
};

struct nbt_occ_s {
    nbt_ctx ctx = nullptr;
    nbt_map_desc desc{};
    size_t nvox = 0;
    float *d_L = nullptr;             // log-odds, dense x-fastest, NaN = never observed (Q36)
    uint32_t *d_flags = nullptr;      // one flag byte per voxel (16-byte padded), zero between calls
    uint32_t *d_list = nullptr;       // flagged voxels of the current cloud (bit 31: hit)
    uint32_t *d_didx = nullptr;       // a2 deltas of the last cloud: dense voxel index ...
    uint16_t *d_dval = nullptr;       // ... and state | level << 8
    int *d_ctl = nullptr;             // per-call control words (kOcc*)
    uint32_t last_points = 0;         // host mirror of the last call's input size
    bool last_filtered = false;
    nbt::DevBuf pts;                  // staged host points
    nbt::DevBuf keys, keys_alt, idx, idx_alt, runs, sorted, filtered, cub_tmp;
    nbt::DevBuf hkeys, hcount, cells;  // hashed voxel filter (integration path)
};

// ------------------------------------------------------------- kernel API

namespace nbt {

// Map store (k_map.cu)
nbt_status launch_map_pack(nbt_ctx ctx, nbt_map m, const uint8_t *d_codes, const uint8_t *d_levels);
nbt_status launch_map_classify(nbt_ctx ctx, const float *d_p, const uint8_t *d_obs, size_t n, double t_occ,
                               double t_free, uint8_t *d_codes_out, uint8_t *d_levels_out);
nbt_status launch_map_update(nbt_ctx ctx, nbt_map m, const int32_t *d_ijk, const uint8_t *d_codes,
                             const uint8_t *d_levels, size_t n);
nbt_status launch_map_unpack(nbt_ctx ctx, nbt_map m, uint8_t *d_codes_out, uint8_t *d_levels_out);

// Perspectives (k_sample.cu)
nbt_status launch_sample(nbt_ctx ctx, const double poi[3], double r_s, int32_t n, uint64_t seed, int32_t mode,
                         double *d_out);

// The ID (k_id.cu)
struct IdLaunch {
    const double *d_persp;   // source perspective array (device)
    int32_t n_src;           // rows in the source array
    int32_t first, stride;   // computed rows: first + i*stride
    int32_t n;               // number of computed rows
    double poi[3];
    nbt_camera cam;
    double range;
    double *d_xyz_out;       // n x 3
    double *d_gain_out;      // n
    uint64_t *d_counts_out;  // n x 4 or null
    int32_t ray_rank = 0, ray_world = 1;      // ray shard (nbt_id_compute_rays)
    uint64_t *d_totals_trace = nullptr;       // ray shard: trace into these n x 5 totals, no finalize
    const uint64_t *d_totals_final = nullptr; // nbt_id_finalize: no trace, finalize these totals
    const GatherDst *gather = nullptr;        // nbt_id_compute_gather: rows to every destination
    int32_t gather_row0 = 0;                  // ... at row gather_row0 + first + i*stride
    const PeerTotals *peer_totals = nullptr;  // nbt_id_compute_rays_gather: counts into every rank
    const PeerTotals *d_peer_totals = nullptr; // ... the same table in device memory
    uint32_t *d_record = nullptr;             // nbt_debug_id_rays: per-ray (U, F, O, L, stop), n x N_E x 5
};
nbt_status launch_id(nbt_ctx ctx, nbt_map m, const IdLaunch &L);
nbt_status launch_debug_trace(nbt_ctx ctx, nbt_map m, const int32_t *d_o, const int32_t *d_e, int32_t n_rays,
                              int32_t max_visits, int32_t *d_ijk, uint8_t *d_code, int32_t *d_len,
                              uint32_t *d_counts, bool wide);
bool debug_needs_wide(const int32_t *o_q16, const int32_t *e_q16, int32_t n_rays);
nbt_status launch_debug_frames(nbt_ctx ctx, nbt_map m, const double poi[3], const double *d_persp, int32_t n,
                               const nbt_camera &cam, double range, int32_t *d_frames);

// IDW (k_idw.cu).  The ring state lives on the device (nbt_idbuf_s::d_meta) so that a
// captured graph replays pushes and queries correctly.
nbt_status launch_idbuf_push(nbt_ctx ctx, nbt_idbuf_s *b, const double *d_xyz, const double *d_gain, int32_t n);
nbt_status launch_idw(nbt_ctx ctx, const nbt_idbuf_s *b, const double *d_q, int32_t n_q, double power_p,
                      double zero_eps, int32_t normalize, double *d_out, int32_t knn = 0);
struct InfoCostArgs {
    const double *pos, *axis;
    int32_t n_traj, per;
    double poi[3];
    double cos_cut, w_i, eps;
    double *o_out, *g_out, *c_out;   // device; o/g may be null
};
nbt_status launch_info_cost(nbt_ctx ctx, const nbt_idbuf_s *b, const InfoCostArgs &a, double power_p,
                            double zero_eps, int32_t normalize);

// Map integration (k_integrate.cu).  d_ctl words of an occupancy store:
enum : int { kOccBad = 0, kOccRays = 1, kOccTouched = 2, kOccDeltas = 3, kOccValid = 4, kOccCtlInts = 8 };
nbt_status launch_voxel_filter(nbt_ctx ctx, nbt_occ_s *o, const double *d_pts, uint32_t n, double leaf,
                               int32_t *d_count_out);
nbt_status launch_integrate(nbt_ctx ctx, nbt_occ_s *o, nbt_map m, const double sensor[3], const double *d_pts,
                            uint32_t n, const nbt_integrate_params &p);

}  // namespace nbt
