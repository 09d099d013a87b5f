// libnbt runtime: the C ABI of include/nbt.h (handles, validation, staging of host
// inputs/outputs, stream ordering).  All arithmetic of the method runs in the kernels
// of k_map.cu, k_sample.cu, k_id.cu and k_idw.cu; this file only moves data and checks
// arguments.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "nbt_internal.cuh"

namespace nbt {

static thread_local std::string g_last_error;
thread_local bool g_capturing = false;

void set_error(const std::string &msg) { g_last_error = msg; }

nbt_status fail(nbt_status s, const std::string &msg)
{
    g_last_error = msg;
    return s;
}

nbt_status cuda_fail(cudaError_t e, const char *what)
{
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return e == cudaErrorMemoryAllocation ? NBT_ERR_OUT_OF_MEMORY : NBT_ERR_CUDA;
}

nbt_status DevBuf::ensure(size_t bytes)
{
    if (bytes <= cap && p) return NBT_OK;
    if (g_capturing) return fail(NBT_ERR_STATE, "a scratch buffer would grow during graph capture: run the "
                                                "sequence once before capturing");
    size_t want = bytes < 256 ? 256 : bytes;
    want = want + want / 4;
    if (p) {
        NBT_CUDA(cudaFree(p));   // implicit device synchronisation: no in-flight user
        p = nullptr;
        cap = 0;
    }
    NBT_CUDA(cudaMalloc(&p, want));
    cap = want;
    return NBT_OK;
}

void DevBuf::release()
{
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

nbt_status HostStage::acquire(size_t bytes)
{
    if (pending) {
        NBT_CUDA(cudaEventSynchronize(ev));
        pending = false;
    }
    if (!ev) NBT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (bytes <= cap && p) return NBT_OK;
    if (p) NBT_CUDA(cudaFreeHost(p));
    p = nullptr;
    size_t want = bytes < 4096 ? 4096 : bytes + bytes / 4;
    NBT_CUDA(cudaHostAlloc(&p, want, cudaHostAllocDefault));
    cap = want;
    return NBT_OK;
}

nbt_status HostStage::mark(cudaStream_t s)
{
    NBT_CUDA(cudaEventRecord(ev, s));
    pending = true;
    return NBT_OK;
}

void HostStage::release()
{
    if (pending && ev) cudaEventSynchronize(ev);
    if (p) cudaFreeHost(p);
    if (ev) cudaEventDestroy(ev);
    p = nullptr;
    ev = nullptr;
    cap = 0;
    pending = false;
}

// Host copies into and out of the pinned stages.  One memcpy thread moves ~10 GB/s, so a
// large input (a 640x576 depth frame is 8.8 MB) is copied by a few persistent worker threads
// in chunks, and the caller issues each chunk's DMA as soon as the chunk is staged: the host
// copy, the PCIe transfer and the workers overlap.  NBT_COPY_THREADS sets the number of
// workers (default 4 on hosts with >= 8 hardware threads; 0 = plain memcpy on the caller).
class CopyPool {
public:
    static CopyPool &get()
    {
        static CopyPool *pool = new CopyPool();   // never destroyed: idle workers end with the process
        return *pool;
    }
    static constexpr size_t kChunk = 512u << 10;
    static constexpr size_t kMinParallel = 1u << 20;

    // Copy src -> dst; on_chunk(offset, len) is called on the caller's thread for every
    // chunk, in order, as soon as that chunk has landed.
    template <typename F>
    void copy(void *dst, const void *src, size_t bytes, bool parallel, F &&on_chunk)
    {
        if (!parallel || workers_.empty() || bytes < kMinParallel) {
            memcpy(dst, src, bytes);
            on_chunk(0, bytes);
            return;
        }
        std::lock_guard<std::mutex> caller(call_mu_);
        const size_t n_chunks = (bytes + kChunk - 1) / kChunk;
        if (done_.size() < n_chunks) {
            std::vector<std::atomic<uint32_t>> fresh(n_chunks);
            done_.swap(fresh);
        }
        for (size_t i = 0; i < n_chunks; ++i) done_[i].store(0, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char *>(dst);
            src_ = static_cast<const char *>(src);
            bytes_ = bytes;
            n_chunks_ = n_chunks;
            next_.store(0, std::memory_order_relaxed);
            active_ = (int)workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        for (size_t i = 0; i < n_chunks; ++i) {
            while (done_[i].load(std::memory_order_acquire) == 0) std::this_thread::yield();
            const size_t off = i * kChunk;
            on_chunk(off, bytes - off < kChunk ? bytes - off : kChunk);
        }
        std::unique_lock<std::mutex> lk(mu_);        // workers are done with dst/src
        idle_cv_.wait(lk, [&] { return active_ == 0; });
    }
    void copy(void *dst, const void *src, size_t bytes, bool parallel)
    {
        copy(dst, src, bytes, parallel, [](size_t, size_t) {});
    }

private:
    CopyPool()
    {
        for (int k = 0; k < kWorkers; ++k) workers_.emplace_back([this] { run(); });
    }
    static constexpr int kWorkers = 4;
    void run()
    {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
            }
            for (;;) {
                const size_t i = next_.fetch_add(1, std::memory_order_relaxed);
                if (i >= n_chunks_) break;
                const size_t off = i * kChunk;
                memcpy(dst_ + off, src_ + off, bytes_ - off < kChunk ? bytes_ - off : kChunk);
                done_[i].store(1, std::memory_order_release);
            }
            std::lock_guard<std::mutex> lk(mu_);
            if (--active_ == 0) idle_cv_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::vector<std::atomic<uint32_t>> done_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, idle_cv_;
    char *dst_ = nullptr;
    const char *src_ = nullptr;
    size_t bytes_ = 0, n_chunks_ = 0;
    std::atomic<size_t> next_{0};
    int active_ = 0;
    uint64_t gen_ = 0;
};

// Copy a host array into device scratch through a pinned stage (async, stream-ordered).
static nbt_status stage_h2d(nbt_ctx ctx, HostStage &st, DevBuf &dst, const void *src, size_t bytes)
{
    nbt_status s;
    if ((s = dst.ensure(bytes))) return s;
    if (bytes == 0) return NBT_OK;
    if (ctx->opt.h2d_mode == 1) {   // experiment: let the driver stage the pageable source
        NBT_CUDA(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        return NBT_OK;
    }
    if ((s = st.acquire(bytes))) return s;
    cudaError_t e = cudaSuccess;
    CopyPool::get().copy(st.p, src, bytes, ctx->opt.copy_threads > 0, [&](size_t off, size_t len) {
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(static_cast<char *>(dst.p) + off, static_cast<char *>(st.p) + off, len,
                                cudaMemcpyHostToDevice, ctx->stream);
    });
    if (e != cudaSuccess) return cuda_fail(e, "stage_h2d");
    return st.mark(ctx->stream);
}

// Copy device results to a host buffer (synchronises the stream).
static nbt_status d2h_sync(nbt_ctx ctx, void *dst, const void *src, size_t bytes)
{
    if (bytes == 0) return NBT_OK;
    nbt_status s;
    if ((s = ctx->stage_out.acquire(bytes))) return s;
    NBT_CUDA(cudaMemcpyAsync(ctx->stage_out.p, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    CopyPool::get().copy(dst, ctx->stage_out.p, bytes, ctx->opt.copy_threads > 0);
    return NBT_OK;
}

static nbt_status bind(nbt_ctx ctx)
{
    if (!ctx) return fail(NBT_ERR_INVALID_ARG, "null ctx");
    NBT_CUDA(cudaSetDevice(ctx->device));
    return NBT_OK;
}

// Device-side validation status recorded since the last sync.
static nbt_status take_device_error(nbt_ctx ctx, const char *where)
{
    NBT_CUDA(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    int e = *ctx->h_err;
    if (e != 0) {
        NBT_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
        NBT_CUDA(cudaStreamSynchronize(ctx->stream));
        return fail((nbt_status)e, std::string(where) + ": device-side validation failed (" +
                                       nbt_status_string((nbt_status)e) + ")");
    }
    return NBT_OK;
}

cudaEvent_t Profiler::take()
{
    cudaEvent_t e = nullptr;
    if (!pool.empty()) {
        e = pool.back();
        pool.pop_back();
    } else if (cudaEventCreate(&e) != cudaSuccess) {
        e = nullptr;
    }
    return e;
}

ProfScope::ProfScope(nbt_ctx c, int k) : ctx(c), kernel(k)
{
    if (!ctx->prof.on || !((ctx->prof.mask >> k) & 1u)) return;
    if (ctx->capturing) {
        // a fresh event owned by the graph; recorded as an event node at every replay
        if (cudaEventCreate(&start) != cudaSuccess) start = nullptr;
        if (start) cudaEventRecordWithFlags(start, ctx->stream, cudaEventRecordExternal);
        return;
    }
    start = ctx->prof.take();
    if (start) cudaEventRecord(start, ctx->stream);
}

ProfScope::~ProfScope()
{
    if (!start) return;
    if (ctx->capturing) {
        cudaEvent_t end = nullptr;
        if (cudaEventCreate(&end) == cudaSuccess) {
            cudaEventRecordWithFlags(end, ctx->stream, cudaEventRecordExternal);
            ctx->cap_pairs.push_back(CapPair{kernel, start, end});
        } else {
            cudaEventDestroy(start);
        }
        return;
    }
    cudaEvent_t end = ctx->prof.take();
    if (!end) {
        ctx->prof.pool.push_back(start);
        return;
    }
    cudaEventRecord(end, ctx->stream);
    ctx->prof.pending[kernel].emplace_back(start, end);
}

static bool finite3(const double *p) { return isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]); }

// The ctx is released when nbt_ctx_destroy has been called AND every map, ID buffer and
// graph created on it has been destroyed (handles may be destroyed in any order).
static void ctx_free(nbt_ctx ctx)
{
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    DevBuf *bufs[] = {&ctx->persp, &ctx->frames, &ctx->totals, &ctx->counter, &ctx->out_tmp, &ctx->deltas,
                      &ctx->keys, &ctx->keys_alt, &ctx->cub_tmp, &ctx->queries, &ctx->qout, &ctx->idw_tmp, &ctx->poses, &ctx->dbg, &ctx->idw_done};
    for (DevBuf *b : bufs) b->release();
    for (auto &st : ctx->stage_in) st.release();
    for (auto &v : ctx->prof.pending)
        for (auto &pr : v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    for (cudaEvent_t e : ctx->prof.pool) cudaEventDestroy(e);
    ctx->stage_out.release();
    if (ctx->d_err) cudaFree(ctx->d_err);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

static void ctx_retain(nbt_ctx ctx) { ctx->refs++; }

static void ctx_release(nbt_ctx ctx)
{
    if (--ctx->refs == 0) ctx_free(ctx);
}


}  // namespace nbt

using namespace nbt;

extern "C" {

int nbt_abi_version(void) { return NBT_ABI_VERSION; }

const char *nbt_status_string(nbt_status s)
{
    switch (s) {
    case NBT_OK: return "NBT_OK";
    case NBT_ERR_INVALID_ARG: return "NBT_ERR_INVALID_ARG";
    case NBT_ERR_DEGENERATE: return "NBT_ERR_DEGENERATE";
    case NBT_ERR_EMPTY: return "NBT_ERR_EMPTY";
    case NBT_ERR_OUT_OF_MEMORY: return "NBT_ERR_OUT_OF_MEMORY";
    case NBT_ERR_CUDA: return "NBT_ERR_CUDA";
    case NBT_ERR_NCCL: return "NBT_ERR_NCCL";
    case NBT_ERR_STATE: return "NBT_ERR_STATE";
    }
    return "NBT_ERR_UNKNOWN";
}

const char *nbt_last_error_message(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ context

nbt_status nbt_ctx_create(int device, void *cuda_stream, nbt_ctx *out)
{
    if (!out) return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_create: null out");
    *out = nullptr;
    int ndev = 0;
    NBT_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_create: no such device");
    NBT_CUDA(cudaSetDevice(device));
    nbt_ctx c = new (std::nothrow) nbt_ctx_s();
    if (!c) return fail(NBT_ERR_OUT_OF_MEMORY, "nbt_ctx_create");
    c->device = device;
    c->opt.copy_threads = std::thread::hardware_concurrency() >= 8 ? 1 : 0;
    cudaError_t e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess && cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else if (e == cudaSuccess) {
        e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        c->own_stream = true;
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->d_err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaHostAlloc(&c->h_err, sizeof(int), cudaHostAllocDefault);
    if (e != cudaSuccess) {
        nbt_ctx_destroy(c);
        return cuda_fail(e, "nbt_ctx_create");
    }
    *out = c;
    return NBT_OK;
}

// Tuning options (nbt.h): value ranges; none of them changes a result.
nbt_status nbt_ctx_set_option(nbt_ctx ctx, int32_t option, int64_t value)
{
    if (!ctx) return fail(NBT_ERR_INVALID_ARG, "null ctx");
    auto in = [&](int64_t lo, int64_t hi) { return value >= lo && value <= hi; };
    NbtOptions &o = ctx->opt;
    switch (option) {
    case NBT_OPT_TRACE_REFILL_MIN:
        if (!in(1, 32)) break;
        o.refill_min = (int)value;
        return NBT_OK;
    case NBT_OPT_TRACE_CHUNK_MIN:
        if (!in(32, 1024)) break;
        o.chunk_min = (int)((value + 31) / 32 * 32);
        return NBT_OK;
    case NBT_OPT_TRACE_CARVEOUT:
        if (!in(-1, 100)) break;
        o.carveout = (int)value;
        ctx->trace_blocks_per_sm = 0;     // re-apply the carveout and re-read the occupancy
        return NBT_OK;
    case NBT_OPT_DELTA_SORT:
        if (!in(0, 1)) break;
        o.delta_sort = (int)value;
        return NBT_OK;
    case NBT_OPT_FILTER_SORT:
        if (!in(0, 1)) break;
        o.filter_sort = (int)value;
        return NBT_OK;
    case NBT_OPT_H2D_MODE:
        if (!in(0, 1)) break;
        o.h2d_mode = (int)value;
        return NBT_OK;
    case NBT_OPT_COPY_THREADS:
        if (!in(0, 1)) break;
        o.copy_threads = (int)value;
        return NBT_OK;
    case NBT_OPT_WALK_WIDTH:
        if (value != 0 && value != 32 && value != 64) break;
        o.walk_width = (int)value;
        return NBT_OK;
    case NBT_OPT_VERBOSE:
        if (!in(0, 1)) break;
        o.verbose = (int)value;
        ctx->trace_blocks_per_sm = 0;
        return NBT_OK;
    default:
        return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_set_option: unknown option " + std::to_string(option));
    }
    return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_set_option: value " + std::to_string(value) + " out of range for option " +
                                         std::to_string(option));
}

nbt_status nbt_ctx_get_option(nbt_ctx ctx, int32_t option, int64_t *value)
{
    if (!ctx || !value) return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_get_option: null argument");
    const NbtOptions &o = ctx->opt;
    switch (option) {
    case NBT_OPT_TRACE_REFILL_MIN: *value = o.refill_min; return NBT_OK;
    case NBT_OPT_TRACE_CHUNK_MIN: *value = o.chunk_min; return NBT_OK;
    case NBT_OPT_TRACE_CARVEOUT: *value = o.carveout; return NBT_OK;
    case NBT_OPT_DELTA_SORT: *value = o.delta_sort; return NBT_OK;
    case NBT_OPT_FILTER_SORT: *value = o.filter_sort; return NBT_OK;
    case NBT_OPT_H2D_MODE: *value = o.h2d_mode; return NBT_OK;
    case NBT_OPT_COPY_THREADS: *value = o.copy_threads; return NBT_OK;
    case NBT_OPT_WALK_WIDTH: *value = o.walk_width; return NBT_OK;
    case NBT_OPT_VERBOSE: *value = o.verbose; return NBT_OK;
    default: return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_get_option: unknown option " + std::to_string(option));
    }
}

nbt_status nbt_ctx_set_stream(nbt_ctx ctx, void *cuda_stream)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->own_stream) {
        cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
    }
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
    } else {
        NBT_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    return NBT_OK;
}

nbt_status nbt_ctx_sync(nbt_ctx ctx)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_ctx_sync during graph capture");
    return take_device_error(ctx, "nbt_ctx_sync");
}

uint64_t nbt_ctx_launch_count(nbt_ctx ctx) { return ctx ? ctx->launches : 0; }

nbt_status nbt_ctx_capture_begin(nbt_ctx ctx)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_ctx_capture_begin: already capturing");
    NBT_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    ctx->capturing = true;
    g_capturing = true;
    ctx->cap_pairs.clear();
    ctx->cap_launches0 = ctx->launches;
    return NBT_OK;
}

nbt_status nbt_ctx_capture_end(nbt_ctx ctx, nbt_graph *out)
{
    nbt_status s;
    if (!out) return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_capture_end: null out");
    *out = nullptr;
    if ((s = bind(ctx))) return s;
    if (!ctx->capturing) return fail(NBT_ERR_STATE, "nbt_ctx_capture_end: not capturing");
    ctx->capturing = false;
    g_capturing = false;
    nbt_graph g = new (std::nothrow) nbt_graph_s();
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (e != cudaSuccess || !g) {
        delete g;
        for (auto &p : ctx->cap_pairs) { cudaEventDestroy(p.start); cudaEventDestroy(p.end); }
        ctx->cap_pairs.clear();
        return e != cudaSuccess ? cuda_fail(e, "nbt_ctx_capture_end") : fail(NBT_ERR_OUT_OF_MEMORY, "graph");
    }
    g->ctx = ctx;
    ctx_retain(ctx);
    g->graph = graph;
    g->pairs.swap(ctx->cap_pairs);
    g->kernels = ctx->launches - ctx->cap_launches0;
    ctx->launches = ctx->cap_launches0;            // recorded, not launched
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (e != cudaSuccess) {
        nbt_graph_destroy(g);
        return cuda_fail(e, "cudaGraphInstantiate");
    }
    *out = g;
    return NBT_OK;
}

nbt_status nbt_graph_launch(nbt_graph g)
{
    nbt_status s;
    if (!g) return fail(NBT_ERR_INVALID_ARG, "nbt_graph_launch: null graph");
    if ((s = bind(g->ctx))) return s;
    NBT_CUDA(cudaGraphLaunch(g->exec, g->ctx->stream));
    g->ctx->launches += g->kernels;
    return NBT_OK;
}

nbt_status nbt_graph_profile_read(nbt_graph g, int32_t kernel, double *total_ms, uint64_t *launches)
{
    nbt_status s;
    if (!g || !total_ms || !launches) return fail(NBT_ERR_INVALID_ARG, "nbt_graph_profile_read: bad argument");
    if ((s = bind(g->ctx))) return s;
    NBT_CUDA(cudaStreamSynchronize(g->ctx->stream));
    double ms = 0.0;
    uint64_t n = 0;
    for (auto &p : g->pairs) {
        if (p.kernel != kernel) continue;
        float t = 0.f;
        NBT_CUDA(cudaEventElapsedTime(&t, p.start, p.end));
        ms += t;
        ++n;
    }
    *total_ms = ms;
    *launches = n;
    return NBT_OK;
}

void nbt_graph_destroy(nbt_graph g)
{
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    for (auto &p : g->pairs) { cudaEventDestroy(p.start); cudaEventDestroy(p.end); }
    nbt_ctx ctx = g->ctx;
    delete g;
    ctx_release(ctx);
}

nbt_status nbt_ctx_set_profiling(nbt_ctx ctx, int enable)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    ctx->prof.on = enable != 0;
    ctx->prof.mask = ~0u;
    return NBT_OK;
}

nbt_status nbt_ctx_set_profiling_mask(nbt_ctx ctx, uint32_t kernel_mask)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    ctx->prof.on = kernel_mask != 0;
    ctx->prof.mask = kernel_mask;
    return NBT_OK;
}

nbt_status nbt_ctx_profile_read(nbt_ctx ctx, int32_t kernel, double *total_ms, uint64_t *launches, int reset)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (kernel < 0 || kernel >= NBT_KERNEL_COUNT || !total_ms || !launches)
        return fail(NBT_ERR_INVALID_ARG, "nbt_ctx_profile_read: bad argument");
    Profiler &P = ctx->prof;
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto &pr : P.pending[kernel]) {
        float ms = 0.f;
        NBT_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
        P.ms[kernel] += ms;
        P.n[kernel] += 1;
        P.pool.push_back(pr.first);
        P.pool.push_back(pr.second);
    }
    P.pending[kernel].clear();
    *total_ms = P.ms[kernel];
    *launches = P.n[kernel];
    if (reset) {
        P.ms[kernel] = 0;
        P.n[kernel] = 0;
    }
    return NBT_OK;
}

void nbt_ctx_destroy(nbt_ctx ctx)
{
    if (!ctx || ctx->closed) return;
    ctx->closed = true;
    ctx_release(ctx);
}

// --------------------------------------------------------------------- map

void nbt_map_desc_default(nbt_map_desc *d, int32_t nx, int32_t ny, int32_t nz, double voxel_size)
{
    if (!d) return;
    memset(d, 0, sizeof *d);
    d->nx = nx; d->ny = ny; d->nz = nz;
    d->voxel_size = voxel_size;
    d->gain[0] = 1.0;     // Unknown (Eq. 2)
    d->gain[1] = 0.12;    // Free: P = P_min (S:92 clamp, Q15)
    d->gain[2] = 0.03;    // Occupied: 1 - P_max (S:92 clamp, Q15)
    d->outside_policy = NBT_OUTSIDE_UNKNOWN;
    d->layout = NBT_LAYOUT_LINEAR;
    d->state_bits = 2;
}

static nbt_status check_desc(const nbt_map_desc *d)
{
    if (!d) return fail(NBT_ERR_INVALID_ARG, "null map desc");
    if (d->nx < 1 || d->ny < 1 || d->nz < 1 || d->nx > 16384 || d->ny > 16384 || d->nz > 16384)
        return fail(NBT_ERR_INVALID_ARG, "map extents must be in [1, 16384]");
    uint64_t pad = (uint64_t)(d->nx + 2 * kBorder) * (d->ny + 2 * kBorder) * (d->nz + 2 * kBorder);
    if (pad >= (1ull << 32)) return fail(NBT_ERR_INVALID_ARG, "(nx+32)(ny+32)(nz+32) must be < 2^32");
    // the walk addresses the linear 2-bit store by the 32-bit bit offset 2i of a code (k_id.cu)
    if (d->state_bits == 2 && d->layout == NBT_LAYOUT_LINEAR && pad >= (1ull << 31))
        return fail(NBT_ERR_INVALID_ARG, "2-bit linear store: (nx+32)(ny+32)(nz+32) must be < 2^31");
    if (!(d->voxel_size > 0) || !isfinite(d->voxel_size)) return fail(NBT_ERR_INVALID_ARG, "voxel_size must be > 0");
    if (!finite3(d->origin)) return fail(NBT_ERR_INVALID_ARG, "origin must be finite");
    for (int k = 0; k < 3; ++k)
        if (!(d->gain[k] >= 0) || !isfinite(d->gain[k])) return fail(NBT_ERR_INVALID_ARG, "gain must be finite, >= 0");
    if (d->outside_policy != NBT_OUTSIDE_UNKNOWN && d->outside_policy != NBT_OUTSIDE_CLIP)
        return fail(NBT_ERR_INVALID_ARG, "bad outside_policy");
    if (d->layout != NBT_LAYOUT_LINEAR && d->layout != NBT_LAYOUT_MORTON)
        return fail(NBT_ERR_INVALID_ARG, "bad layout");
    if (d->state_bits != 2 && d->state_bits != 8) return fail(NBT_ERR_INVALID_ARG, "state_bits must be 2 or 8");
    return NBT_OK;
}

#ifndef NBT_BANK_PAD
#define NBT_BANK_PAD 1     // 0: rows of nx + 2 kBorder voxels, planes of (nx + 2B)(ny + 2B) (A/B builds)
#endif
static nbt_status map_create(nbt_ctx ctx, const nbt_map_desc *desc, int vbits, bool prob, nbt_map *out)
{
    nbt_status s;
    if (!out) return fail(NBT_ERR_INVALID_ARG, "nbt_map_create: null out");
    *out = nullptr;
    if ((s = bind(ctx)) || (s = check_desc(desc))) return s;
    nbt_map m = new (std::nothrow) nbt_map_s();
    if (!m) return fail(NBT_ERR_OUT_OF_MEMORY, "nbt_map_create");
    m->ctx = ctx;
    ctx_retain(ctx);
    m->desc = *desc;
    m->vbits = vbits;
    m->prob = prob;
    m->px = desc->nx + 2 * kBorder; m->py = desc->ny + 2 * kBorder; m->pz = desc->nz + 2 * kBorder;
#if NBT_BANK_PAD
    if (desc->layout != NBT_LAYOUT_MORTON) {
        // Extra sentinel columns / rows so that neighbouring rows fall into different L1 banks
        // (4-byte banks, 32 of them): a row is an odd number of words (y step = sy words) and a
        // plane is 17 words mod 32 (z step), so a warp's rays spread over a few rows and planes
        // hit distinct banks instead of the plane-aligned same bank (D: px = 544 = 34 words,
        // a plane 18496 words = 0 mod 32).  Skipped when it would break the 2^31 / 2^32 bound.
        const uint32_t per = vbits == 2 ? 16 : 4;
        uint32_t px = (m->px + per - 1) / per * per;
        if (((px / per) & 1u) == 0) px += per;
        const uint32_t sy = (px / per) & 31u;                      // odd
        uint32_t inv = 1;
        while ((sy * inv & 31u) != 1u) inv += 2;                   // sy^-1 mod 32
        const uint32_t want = (17u * inv) & 31u;                   // py = want (mod 32)
        const uint32_t py = m->py + ((want - (m->py & 31u)) & 31u);
        const uint64_t nv = (uint64_t)px * py * m->pz;
        if (nv < (vbits == 2 ? (1ull << 31) : (1ull << 32))) { m->px = px; m->py = py; }
    }
#endif
    m->nvox_pad = (uint64_t)m->px * m->py * m->pz;
    // Store layout (desc->layout): linear by default (fewest instructions per voxel step,
    // fastest on configs C' and D, profiles/r01_layouts.md), or the Morton cube (side >= max
    // extent + 2 kBorder, a power of two, at most 1024^3 voxels and 8x the linear store),
    // which is slightly faster on sparse ray lattices (config B).
    if (desc->layout == NBT_LAYOUT_MORTON) {
        int maxn = desc->nx > desc->ny ? desc->nx : desc->ny;
        maxn = maxn > desc->nz ? maxn : desc->nz;
        int pb = 4;
        while ((1 << pb) < maxn + 2 * kBorder) ++pb;
        uint64_t cube = 1ull << (3 * pb);
        if (pb > 10 || cube > 8 * m->nvox_pad) {
            nbt_map_destroy(m);
            return fail(NBT_ERR_INVALID_ARG, "nbt_map_create: the Morton cube must fit 1024^3 voxels and 8x the linear store");
        }
        m->layout = kLayoutMorton;
        m->pbits = pb;
        m->nvox_pad = cube;
    }
    const size_t per_word = vbits == 2 ? 16 : 4;
    m->nwords = (size_t)((m->nvox_pad + per_word - 1) / per_word);
    cudaError_t e = cudaMalloc(&m->d_words, m->nwords * 4);
    if (e != cudaSuccess) {
        nbt_map_destroy(m);
        return cuda_fail(e, "nbt_map_create: cudaMalloc");
    }
    // all Unknown inside, sentinel ring outside: pack from a null code array
    DevBuf zeros;
    size_t n = (size_t)desc->nx * desc->ny * desc->nz;
    if ((s = zeros.ensure(n))) { nbt_map_destroy(m); return s; }
    e = cudaMemsetAsync(zeros.p, 0, n, ctx->stream);
    if (e == cudaSuccess) s = launch_map_pack(ctx, m, zeros.as<uint8_t>(), nullptr);
    else s = cuda_fail(e, "nbt_map_create: memset");
    if (s == NBT_OK) {
        e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) s = cuda_fail(e, "nbt_map_create: sync");
    }
    zeros.release();
    if (s) { nbt_map_destroy(m); return s; }
    *out = m;
    return NBT_OK;
}

// Bits per voxel of a state-only map (desc->state_bits): 2 (packed codes, default) or 8
// (one byte per voxel: no rotate per visit, 4x the bytes).
nbt_status nbt_map_create(nbt_ctx ctx, const nbt_map_desc *desc, nbt_map *out)
{
    return map_create(ctx, desc, desc ? desc->state_bits : 2, false, out);
}

nbt_status nbt_map_create_prob(nbt_ctx ctx, const nbt_map_desc *desc, nbt_map *out)
{
    return map_create(ctx, desc, 8, true, out);
}

static nbt_status map_nvox(nbt_map m, size_t n, const char *who)
{
    if (!m) return fail(NBT_ERR_INVALID_ARG, std::string(who) + ": null map");
    size_t want = (size_t)m->desc.nx * m->desc.ny * m->desc.nz;
    if (n != want) return fail(NBT_ERR_INVALID_ARG, std::string(who) + ": n must be nx*ny*nz");
    return NBT_OK;
}

nbt_status nbt_map_upload(nbt_map m, const uint8_t *codes, size_t n, int on_device)
{
    nbt_status s;
    if ((s = map_nvox(m, n, "nbt_map_upload"))) return s;
    nbt_ctx ctx = m->ctx;
    if ((s = bind(ctx))) return s;
    if (!codes) return fail(NBT_ERR_INVALID_ARG, "nbt_map_upload: null codes");
    if ((s = take_device_error(ctx, "nbt_map_upload (earlier work)"))) return s;
    const uint8_t *src = codes;
    DevBuf tmp;
    if (!on_device) {
        for (size_t i = 0; i < n; ++i)
            if (codes[i] > 2) return fail(NBT_ERR_INVALID_ARG, "nbt_map_upload: code >= 3 at " + std::to_string(i));
        if ((s = tmp.ensure(n))) return s;
        cudaError_t e = cudaMemcpyAsync(tmp.p, codes, n, cudaMemcpyHostToDevice, ctx->stream);
        if (e != cudaSuccess) { tmp.release(); return cuda_fail(e, "nbt_map_upload: H2D"); }
        src = tmp.as<uint8_t>();
    }
    s = launch_map_pack(ctx, m, src, nullptr);
    if (s == NBT_OK) s = take_device_error(ctx, "nbt_map_upload");
    tmp.release();
    return s;
}

nbt_status nbt_map_upload_prob(nbt_map m, const float *p, const uint8_t *observed, size_t n, int on_device,
                               double t_occ, double t_free)
{
    nbt_status s;
    if ((s = map_nvox(m, n, "nbt_map_upload_prob"))) return s;
    nbt_ctx ctx = m->ctx;
    if ((s = bind(ctx))) return s;
    if (!p || !observed) return fail(NBT_ERR_INVALID_ARG, "nbt_map_upload_prob: null input");
    if (!isfinite(t_occ) || !isfinite(t_free)) return fail(NBT_ERR_INVALID_ARG, "thresholds must be finite");
    DevBuf dp, dobs, codes, levels;
    const float *sp = p;
    const uint8_t *so = observed;
    cudaError_t e = cudaSuccess;
    if (!on_device) {
        if ((s = dp.ensure(n * 4)) || (s = dobs.ensure(n))) return s;
        e = cudaMemcpyAsync(dp.p, p, n * 4, cudaMemcpyHostToDevice, ctx->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dobs.p, observed, n, cudaMemcpyHostToDevice, ctx->stream);
        sp = dp.as<float>();
        so = dobs.as<uint8_t>();
    }
    const bool prob = m->prob;
    if (e == cudaSuccess && (s = codes.ensure(n)) == NBT_OK && (!prob || (s = levels.ensure(n)) == NBT_OK)) {
        s = launch_map_classify(ctx, sp, so, n, t_occ, t_free, codes.as<uint8_t>(),
                                prob ? levels.as<uint8_t>() : nullptr);
        if (s == NBT_OK) s = launch_map_pack(ctx, m, codes.as<uint8_t>(), prob ? levels.as<uint8_t>() : nullptr);
        if (s == NBT_OK) s = take_device_error(ctx, "nbt_map_upload_prob");
    } else if (e != cudaSuccess) {
        s = cuda_fail(e, "nbt_map_upload_prob: H2D");
    }
    cudaStreamSynchronize(ctx->stream);
    dp.release(); dobs.release(); codes.release(); levels.release();
    return s;
}

nbt_status nbt_map_update(nbt_map m, const int32_t *ijk, const uint8_t *codes, size_t n, int on_device)
{
    if (!m) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update: null map");
    nbt_ctx ctx = m->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (n == 0) return NBT_OK;
    if (!ijk || !codes) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update: null input");
    const int32_t *dijk = ijk;
    const uint8_t *dcodes = codes;
    if (ctx->capturing && !on_device) return fail(NBT_ERR_STATE, "nbt_map_update: host deltas during graph capture");
    if (!on_device) {
        for (size_t i = 0; i < n; ++i) {
            const int32_t *v = ijk + 3 * i;
            if (v[0] < 0 || v[1] < 0 || v[2] < 0 || v[0] >= m->desc.nx || v[1] >= m->desc.ny || v[2] >= m->desc.nz)
                return fail(NBT_ERR_INVALID_ARG, "nbt_map_update: voxel outside the grid at " + std::to_string(i));
            if (codes[i] > 2) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update: code >= 3 at " + std::to_string(i));
        }
        // one staging area for [ijk | codes]
        size_t bytes = n * 12 + n;
        if ((s = ctx->deltas.ensure(bytes)) || (s = ctx->stage_in[1].acquire(bytes))) return s;
        memcpy(ctx->stage_in[1].p, ijk, n * 12);
        memcpy((char *)ctx->stage_in[1].p + n * 12, codes, n);
        NBT_CUDA(cudaMemcpyAsync(ctx->deltas.p, ctx->stage_in[1].p, bytes, cudaMemcpyHostToDevice, ctx->stream));
        if ((s = ctx->stage_in[1].mark(ctx->stream))) return s;
        dijk = ctx->deltas.as<int32_t>();
        dcodes = ctx->deltas.as<uint8_t>() + n * 12;
    }
    return launch_map_update(ctx, m, dijk, dcodes, nullptr, n);
}

nbt_status nbt_map_update_prob(nbt_map m, const int32_t *ijk, const float *p, const uint8_t *observed, size_t n,
                               int on_device, double t_occ, double t_free)
{
    if (!m) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update_prob: null map");
    nbt_ctx ctx = m->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (n == 0) return NBT_OK;
    if (!ijk || !p || !observed || !isfinite(t_occ) || !isfinite(t_free))
        return fail(NBT_ERR_INVALID_ARG, "nbt_map_update_prob: bad argument");
    if (n >= (1ull << 31)) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update_prob: too many deltas");
    if (ctx->capturing && !on_device)
        return fail(NBT_ERR_STATE, "nbt_map_update_prob: host deltas during graph capture");
    // device scratch: [ijk 12n | p 4n | observed n | codes n | levels n]
    const size_t bytes = n * 19;
    if ((s = ctx->deltas.ensure(bytes))) return s;
    char *base = ctx->deltas.as<char>();
    const int32_t *dijk = ijk;
    const float *dp = p;
    const uint8_t *dobs = observed;
    if (!on_device) {
        for (size_t i = 0; i < n; ++i) {
            const int32_t *v = ijk + 3 * i;
            if (v[0] < 0 || v[1] < 0 || v[2] < 0 || v[0] >= m->desc.nx || v[1] >= m->desc.ny || v[2] >= m->desc.nz)
                return fail(NBT_ERR_INVALID_ARG, "nbt_map_update_prob: voxel outside the grid at " + std::to_string(i));
            if (!isfinite(p[i])) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update_prob: non-finite p");
        }
        if ((s = ctx->stage_in[1].acquire(n * 17))) return s;
        memcpy(ctx->stage_in[1].p, ijk, n * 12);
        memcpy((char *)ctx->stage_in[1].p + n * 12, p, n * 4);
        memcpy((char *)ctx->stage_in[1].p + n * 16, observed, n);
        NBT_CUDA(cudaMemcpyAsync(base, ctx->stage_in[1].p, n * 17, cudaMemcpyHostToDevice, ctx->stream));
        if ((s = ctx->stage_in[1].mark(ctx->stream))) return s;
        dijk = reinterpret_cast<const int32_t *>(base);
        dp = reinterpret_cast<const float *>(base + n * 12);
        dobs = reinterpret_cast<const uint8_t *>(base + n * 16);
    }
    uint8_t *dcodes = reinterpret_cast<uint8_t *>(base + n * 17);
    uint8_t *dlevels = reinterpret_cast<uint8_t *>(base + n * 18);
    if ((s = launch_map_classify(ctx, dp, dobs, n, t_occ, t_free, dcodes, dlevels))) return s;
    return launch_map_update(ctx, m, dijk, dcodes, m->prob ? dlevels : nullptr, n);
}

nbt_status nbt_map_device_buffer(nbt_map m, void **dev_ptr, size_t *bytes)
{
    if (!m || !dev_ptr || !bytes) return fail(NBT_ERR_INVALID_ARG, "nbt_map_device_buffer: null argument");
    *dev_ptr = m->d_words;
    *bytes = m->nwords * 4;
    return NBT_OK;
}

nbt_status nbt_map_download(nbt_map m, uint8_t *codes_out, size_t n)
{
    nbt_status s;
    if ((s = map_nvox(m, n, "nbt_map_download"))) return s;
    if (!codes_out) return fail(NBT_ERR_INVALID_ARG, "nbt_map_download: null out");
    nbt_ctx ctx = m->ctx;
    if ((s = bind(ctx))) return s;
    DevBuf tmp;
    if ((s = tmp.ensure(n))) return s;
    s = launch_map_unpack(ctx, m, tmp.as<uint8_t>(), nullptr);
    if (s == NBT_OK) {
        cudaError_t e = cudaMemcpyAsync(codes_out, tmp.p, n, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) s = cuda_fail(e, "nbt_map_download");
    }
    tmp.release();
    return s;
}

nbt_status nbt_map_download_levels(nbt_map m, uint8_t *levels_out, size_t n)
{
    nbt_status s;
    if ((s = map_nvox(m, n, "nbt_map_download_levels"))) return s;
    if (!levels_out) return fail(NBT_ERR_INVALID_ARG, "nbt_map_download_levels: null out");
    if (!m->prob) return fail(NBT_ERR_STATE, "nbt_map_download_levels: map stores no probabilities");
    nbt_ctx ctx = m->ctx;
    if ((s = bind(ctx))) return s;
    DevBuf tmp;
    if ((s = tmp.ensure(n))) return s;
    s = launch_map_unpack(ctx, m, nullptr, tmp.as<uint8_t>());
    if (s == NBT_OK) {
        cudaError_t e = cudaMemcpyAsync(levels_out, tmp.p, n, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) s = cuda_fail(e, "nbt_map_download_levels");
    }
    tmp.release();
    return s;
}

nbt_status nbt_map_get_desc(nbt_map m, nbt_map_desc *out)
{
    if (!m || !out) return fail(NBT_ERR_INVALID_ARG, "nbt_map_get_desc: null argument");
    *out = m->desc;
    return NBT_OK;
}

void nbt_map_destroy(nbt_map m)
{
    if (!m) return;
    cudaSetDevice(m->ctx->device);
    cudaStreamSynchronize(m->ctx->stream);
    if (m->d_words) cudaFree(m->d_words);
    if (m->d_win) cudaFree(m->d_win);
    nbt_ctx ctx = m->ctx;
    delete m;
    ctx_release(ctx);
}

// ------------------------------------------------------- map integration (f3)

void nbt_integrate_params_default(nbt_integrate_params *p, double voxel_size)
{
    if (!p) return;
    p->p_hit = 0.7; p->p_miss = 0.4;
    p->p_min = 0.12; p->p_max = 0.97;
    p->t_occ = 0.5; p->t_free = 0.5;
    p->max_range = 5.0;
    p->leaf = voxel_size;
}

static void occ_free(nbt_occ_s *o)
{
    for (void *q : {(void *)o->d_L, (void *)o->d_flags, (void *)o->d_list, (void *)o->d_didx, (void *)o->d_dval,
                    (void *)o->d_ctl})
        if (q) cudaFree(q);
    for (DevBuf *b : {&o->pts, &o->keys, &o->keys_alt, &o->idx, &o->idx_alt, &o->runs, &o->sorted, &o->filtered,
                      &o->cub_tmp, &o->hkeys, &o->hcount, &o->cells})
        b->release();
}

nbt_status nbt_occ_create(nbt_ctx ctx, const nbt_map_desc *desc, nbt_occ *out)
{
    nbt_status s;
    if (!out) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_create: null out");
    *out = nullptr;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_occ_create during graph capture");
    if (!desc || desc->nx < 1 || desc->ny < 1 || desc->nz < 1 || !(desc->voxel_size > 0) ||
        !isfinite(desc->voxel_size) || !isfinite(desc->origin[0]) || !isfinite(desc->origin[1]) ||
        !isfinite(desc->origin[2]))
        return fail(NBT_ERR_INVALID_ARG, "nbt_occ_create: bad descriptor");
    const uint64_t nvox = (uint64_t)desc->nx * desc->ny * desc->nz;
    if (nvox >= (1ull << 31)) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_create: grid too large (>= 2^31 voxels)");
    auto *o = new nbt_occ_s;
    o->ctx = ctx;
    o->desc = *desc;
    o->nvox = nvox;
    const size_t nwords = (nvox + 15) / 16 * 4;       // flag bytes, padded to 16-byte groups
    cudaError_t e = cudaMalloc(&o->d_L, nvox * 4);
    if (e == cudaSuccess) e = cudaMalloc(&o->d_flags, nwords * 4);
    if (e == cudaSuccess) e = cudaMalloc(&o->d_list, nvox * 4);
    if (e == cudaSuccess) e = cudaMalloc(&o->d_didx, nvox * 4);
    if (e == cudaSuccess) e = cudaMalloc(&o->d_dval, nvox * 2);
    if (e == cudaSuccess) e = cudaMalloc(&o->d_ctl, kOccCtlInts * sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(o->d_L, 0xff, nvox * 4, ctx->stream);   // 0xffffffff: a NaN
    if (e == cudaSuccess) e = cudaMemsetAsync(o->d_flags, 0, nwords * 4, ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(o->d_ctl, 0, kOccCtlInts * sizeof(int), ctx->stream);
    if (e != cudaSuccess) {
        occ_free(o);
        delete o;
        return e == cudaErrorMemoryAllocation ? fail(NBT_ERR_OUT_OF_MEMORY, "nbt_occ_create: out of device memory")
                                              : cuda_fail(e, "nbt_occ_create");
    }
    ctx_retain(ctx);
    *out = o;
    return NBT_OK;
}

void nbt_occ_destroy(nbt_occ o)
{
    if (!o) return;
    cudaSetDevice(o->ctx->device);
    cudaStreamSynchronize(o->ctx->stream);
    occ_free(o);
    nbt_ctx ctx = o->ctx;
    delete o;
    ctx_release(ctx);
}

nbt_status nbt_occ_upload(nbt_occ o, const float *logodds, size_t n, int on_device)
{
    if (!o || !logodds) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_upload: null argument");
    if (n != o->nvox) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_upload: n must be nx*ny*nz");
    nbt_ctx ctx = o->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing && !on_device) return fail(NBT_ERR_STATE, "nbt_occ_upload: host input during graph capture");
    if (on_device) {
        NBT_CUDA(cudaMemcpyAsync(o->d_L, logodds, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        return NBT_OK;
    }
    NBT_CUDA(cudaMemcpyAsync(o->d_L, logodds, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));   // pageable source: keep it alive until copied
    return NBT_OK;
}

nbt_status nbt_occ_download(nbt_occ o, float *out, size_t n)
{
    if (!o || !out) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_download: null argument");
    if (n != o->nvox) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_download: n must be nx*ny*nz");
    nbt_ctx ctx = o->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_occ_download during graph capture");
    NBT_CUDA(cudaMemcpyAsync(out, o->d_L, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    return NBT_OK;
}

static nbt_status check_integrate_params(const nbt_integrate_params &p)
{
    auto prob = [](double v) { return v > 0.0 && v < 1.0; };
    if (!prob(p.p_hit) || !prob(p.p_miss) || !prob(p.p_min) || !prob(p.p_max) || !(p.p_min <= p.p_max) ||
        !prob(p.t_occ) || !prob(p.t_free) || isnan(p.max_range) || !(p.leaf >= 0.0) || !isfinite(p.leaf))
        return fail(NBT_ERR_INVALID_ARG, "nbt_integrate_params: probabilities must lie in (0,1), p_min <= p_max, "
                                         "leaf >= 0 finite");
    return NBT_OK;
}

nbt_status nbt_occ_integrate(nbt_occ o, nbt_map map, const double sensor[3], const double *points, int64_t n,
                             int on_device, const nbt_integrate_params *prm)
{
    if (!o || !sensor) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_integrate: null argument");
    nbt_ctx ctx = o->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (n < 0 || n >= (1ll << 31)) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_integrate: n out of range");
    if (n > 0 && !points) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_integrate: null points");
    if (!isfinite(sensor[0]) || !isfinite(sensor[1]) || !isfinite(sensor[2]))
        return fail(NBT_ERR_INVALID_ARG, "nbt_occ_integrate: non-finite sensor origin");
    if (map && (map->ctx != ctx || map->desc.nx != o->desc.nx || map->desc.ny != o->desc.ny ||
                map->desc.nz != o->desc.nz))
        return fail(NBT_ERR_STATE, "nbt_occ_integrate: map of another ctx or grid");
    nbt_integrate_params p;
    if (prm) p = *prm;
    else nbt_integrate_params_default(&p, o->desc.voxel_size);
    if ((s = check_integrate_params(p))) return s;
    if (ctx->capturing && !on_device && n > 0)
        return fail(NBT_ERR_STATE, "nbt_occ_integrate: host points during graph capture");
    const double *dpts = points;
    if (!on_device && n > 0) {
        if ((s = stage_h2d(ctx, ctx->stage_in[0], o->pts, points, (size_t)n * 24))) return s;
        dpts = o->pts.as<double>();
    }
    return launch_integrate(ctx, o, map, sensor, dpts, (uint32_t)n, p);
}

nbt_status nbt_occ_stats(nbt_occ o, int64_t out[4])
{
    if (!o || !out) return fail(NBT_ERR_INVALID_ARG, "nbt_occ_stats: null argument");
    nbt_ctx ctx = o->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_occ_stats during graph capture");
    int ctl[kOccCtlInts];
    if ((s = d2h_sync(ctx, ctl, o->d_ctl, sizeof ctl))) return s;
    if ((s = take_device_error(ctx, "nbt_occ_integrate"))) return s;
    out[0] = o->last_points;
    out[1] = o->last_filtered ? (int64_t)(uint32_t)ctl[kOccRays] : (int64_t)o->last_points;
    out[2] = (uint32_t)ctl[kOccTouched];
    out[3] = (uint32_t)ctl[kOccDeltas];
    return NBT_OK;
}

nbt_status nbt_occ_deltas(nbt_occ o, int32_t *ijk, uint8_t *codes, uint8_t *levels, size_t cap, size_t *n_out)
{
    if (!o || !n_out || (cap > 0 && (!ijk || !codes || !levels)))
        return fail(NBT_ERR_INVALID_ARG, "nbt_occ_deltas: null argument");
    nbt_ctx ctx = o->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_occ_deltas during graph capture");
    int ctl[kOccCtlInts];
    if ((s = d2h_sync(ctx, ctl, o->d_ctl, sizeof ctl))) return s;
    const size_t cnt = (uint32_t)ctl[kOccDeltas];
    *n_out = cnt;
    const size_t k = cnt < cap ? cnt : cap;
    if (k == 0) return NBT_OK;
    std::vector<uint32_t> idx(k);
    std::vector<uint16_t> val(k);
    NBT_CUDA(cudaMemcpyAsync(idx.data(), o->d_didx, k * 4, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaMemcpyAsync(val.data(), o->d_dval, k * 2, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint32_t nx = (uint32_t)o->desc.nx, ny = (uint32_t)o->desc.ny;
    for (size_t i = 0; i < k; ++i) {
        const uint32_t v = idx[i];
        ijk[3 * i] = (int32_t)(v % nx);
        ijk[3 * i + 1] = (int32_t)((v / nx) % ny);
        ijk[3 * i + 2] = (int32_t)(v / nx / ny);
        codes[i] = (uint8_t)(val[i] & 0xff);
        levels[i] = (uint8_t)(val[i] >> 8);
    }
    return NBT_OK;
}

nbt_status nbt_voxel_filter(nbt_ctx ctx, const double *points, int64_t n, int on_device, double leaf,
                            double *out_xyz, int32_t *out_count, int64_t *m_out)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (!m_out || n < 0 || n >= (1ll << 31) || (n > 0 && (!points || !out_xyz)) || !(leaf > 0) ||
        !isfinite(leaf))
        return fail(NBT_ERR_INVALID_ARG, "nbt_voxel_filter: bad argument");
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_voxel_filter during graph capture");
    *m_out = 0;
    if (n == 0) return NBT_OK;
    nbt_occ_s tmp;
    tmp.ctx = ctx;
    DevBuf ctl, cnt;
    if ((s = ctl.ensure(kOccCtlInts * sizeof(int))) || (s = cnt.ensure((size_t)n * 4))) return s;
    tmp.d_ctl = ctl.as<int>();
    NBT_CUDA(cudaMemsetAsync(tmp.d_ctl, 0, kOccCtlInts * sizeof(int), ctx->stream));
    const double *dpts = points;
    if (!on_device) {
        if ((s = stage_h2d(ctx, ctx->stage_in[0], tmp.pts, points, (size_t)n * 24))) return s;
        dpts = tmp.pts.as<double>();
    }
    s = launch_voxel_filter(ctx, &tmp, dpts, (uint32_t)n, leaf, cnt.as<int32_t>());
    int c[kOccCtlInts] = {0};
    if (s == NBT_OK) s = d2h_sync(ctx, c, tmp.d_ctl, sizeof c);
    if (s == NBT_OK) s = take_device_error(ctx, "nbt_voxel_filter");
    if (s == NBT_OK) {
        const size_t m = (uint32_t)c[kOccRays];
        cudaError_t e = cudaMemcpyAsync(out_xyz, tmp.filtered.p, m * 24, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess && out_count)
            e = cudaMemcpyAsync(out_count, cnt.p, m * 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) s = cuda_fail(e, "nbt_voxel_filter");
        *m_out = (int64_t)m;
    }
    cudaStreamSynchronize(ctx->stream);
    for (DevBuf *b : {&ctl, &cnt, &tmp.pts, &tmp.keys, &tmp.keys_alt, &tmp.idx, &tmp.idx_alt, &tmp.runs,
                      &tmp.sorted, &tmp.filtered, &tmp.cub_tmp})
        b->release();
    return s;
}

// ------------------------------------------------------------------ camera

nbt_status nbt_camera_from_fov(double fov_h, double fov_v, int32_t w, int32_t h, nbt_camera *out)
{
    if (!out || w < 1 || h < 1 || w > 65535 || h > 65535 || !(fov_h > 0 && fov_h < M_PI) || !(fov_v > 0 && fov_v < M_PI))
        return fail(NBT_ERR_INVALID_ARG, "nbt_camera_from_fov: need 0 < fov < pi and 1 <= w, h <= 65535");
    out->width = w;
    out->height = h;
    out->tan_half_fov_h = tan(fov_h / 2.0);
    out->tan_half_fov_v = tan(fov_v / 2.0);
    out->cx = (w - 1) / 2.0;
    out->cy = (h - 1) / 2.0;
    out->fx = (w > 1) ? (w - 1) / (2.0 * out->tan_half_fov_h) : 1.0;
    out->fy = (h > 1) ? (h - 1) / (2.0 * out->tan_half_fov_v) : 1.0;
    out->add_corners = 0;
    return NBT_OK;
}

nbt_status nbt_camera_from_grid_scaling(double fov_h, double fov_v, double range, double voxel_size, double s_g,
                                        nbt_camera *out)
{
    if (!out || !(range > 0) || !(voxel_size > 0) || !(s_g >= 1.0) || !(fov_h > 0 && fov_h < M_PI) ||
        !(fov_v > 0 && fov_v < M_PI))
        return fail(NBT_ERR_INVALID_ARG, "nbt_camera_from_grid_scaling: bad argument");
    double delta = s_g * voxel_size;
    double th = tan(fov_h / 2.0), tv = tan(fov_v / 2.0);
    double rh = (range * th) / delta, rv = (range * tv) / delta;
    double mh = floor(rh + 1e-9), mv = floor(rv + 1e-9);   // reading Q8: border point kept within 1e-9
    if (mh > 30000 || mv > 30000) return fail(NBT_ERR_INVALID_ARG, "nbt_camera_from_grid_scaling: lattice too large");
    out->width = 2 * (int32_t)mh + 1;
    out->height = 2 * (int32_t)mv + 1;
    out->cx = mh;
    out->cy = mv;
    out->fx = range / delta;
    out->fy = range / delta;
    out->tan_half_fov_h = th;
    out->tan_half_fov_v = tv;
    out->add_corners = !(fabs(rh - mh) <= 1e-9 && fabs(rv - mv) <= 1e-9);   // Q9 dedup
    return NBT_OK;
}

int32_t nbt_camera_num_rays(const nbt_camera *cam)
{
    if (!cam) return 0;
    return cam->width * cam->height + (cam->add_corners ? 4 : 0);
}

static nbt_status check_camera(const nbt_camera *cam)
{
    if (!cam) return fail(NBT_ERR_INVALID_ARG, "null camera");
    if (cam->width < 1 || cam->height < 1 || cam->width > 65535 || cam->height > 65535)
        return fail(NBT_ERR_INVALID_ARG, "camera lattice must be 1..65535 per axis");
    if (!(cam->fx > 0) || !(cam->fy > 0) || !isfinite(cam->fx) || !isfinite(cam->fy))
        return fail(NBT_ERR_INVALID_ARG, "camera fx, fy must be finite and > 0");
    if (cam->cx * 2.0 != cam->width - 1 || cam->cy * 2.0 != cam->height - 1)
        return fail(NBT_ERR_INVALID_ARG, "camera principal point must be the lattice centre (2cx = W-1)");
    if (!isfinite(cam->tan_half_fov_h) || !isfinite(cam->tan_half_fov_v))
        return fail(NBT_ERR_INVALID_ARG, "camera tan_half_fov must be finite");
    if ((int64_t)cam->width * cam->height > (1ll << 30)) return fail(NBT_ERR_INVALID_ARG, "too many rays");
    return NBT_OK;
}

// ------------------------------------------------------------ perspectives

nbt_status nbt_sample_perspectives(nbt_ctx ctx, const double poi[3], double r_s, int32_t n, uint64_t seed,
                                   int32_t mode, double *xyz_out, int out_on_device)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (!poi || !finite3(poi) || !(r_s > 0) || !isfinite(r_s) || n < 0 || (n > 0 && !xyz_out) ||
        (mode != NBT_SAMPLE_BALL && mode != NBT_SAMPLE_SURFACE))
        return fail(NBT_ERR_INVALID_ARG, "nbt_sample_perspectives: bad argument");
    if (n == 0) return NBT_OK;
    if (ctx->capturing && !out_on_device)
        return fail(NBT_ERR_STATE, "nbt_sample_perspectives: host output during graph capture");
    double *dst = xyz_out;
    if (!out_on_device) {
        if ((s = ctx->out_tmp.ensure((size_t)n * 24))) return s;
        dst = ctx->out_tmp.as<double>();
    }
    if ((s = launch_sample(ctx, poi, r_s, n, seed, mode, dst))) return s;
    if (!out_on_device) return d2h_sync(ctx, xyz_out, dst, (size_t)n * 24);
    return NBT_OK;
}

// ----------------------------------------------------------------- the ID

// Ray-shard / split-finalize options of the ID entry points (nbt_id_compute_rays,
// nbt_id_finalize); the defaults are the whole ID.
struct IdExtra {
    int32_t ray_rank = 0, ray_world = 1;
    uint64_t *totals_trace = nullptr;
    const uint64_t *totals_final = nullptr;
    const GatherDst *gather = nullptr;
    int32_t gather_row0 = 0;
    const PeerTotals *peer_totals = nullptr;     // host copy (which ranks)
    const PeerTotals *d_peer_totals = nullptr;   // the same table in device memory
    uint32_t *record = nullptr;                  // nbt_debug_id_rays: per-ray counts (device)
};

// A caller's device array must live on the ctx's device (device or managed memory).
static nbt_status check_device_ptr(nbt_ctx ctx, const void *p, const std::string &what)
{
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(NBT_ERR_INVALID_ARG, what + ": not a device pointer");
    }
    if ((a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) || a.device != ctx->device)
        return fail(NBT_ERR_INVALID_ARG, what + ": must be device memory on the ctx's device");
    return NBT_OK;
}

static nbt_status id_common(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp, int32_t n_persp,
                            int persp_on_device, int32_t first, int32_t stride, const nbt_camera *cam, double range,
                            nbt_ig_cloud *out, const char *who, const IdExtra &x = IdExtra())
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (!m || m->ctx != ctx) return fail(NBT_ERR_STATE, std::string(who) + ": map belongs to another ctx");
    const bool shard = x.totals_trace != nullptr || x.gather != nullptr || x.peer_totals != nullptr;
    if (!poi || !finite3(poi) || (!out && !shard) || n_persp < 0 || !(range > 0) || !isfinite(range))
        return fail(NBT_ERR_INVALID_ARG, std::string(who) + ": bad argument");
    if ((s = check_camera(cam))) return s;
    if (first < 0 || stride < 1) return fail(NBT_ERR_INVALID_ARG, std::string(who) + ": bad first/stride");
    if (ctx->capturing && (!persp_on_device || (!shard && !out->on_device)))
        return fail(NBT_ERR_STATE, std::string(who) + ": host buffers during graph capture");
    int32_t n = (first < n_persp) ? (n_persp - first + stride - 1) / stride : 0;
    if (n == 0) return NBT_OK;
    if (!persp || (!shard && (!out->xyz || !out->gain)))
        return fail(NBT_ERR_INVALID_ARG, std::string(who) + ": null buffer");
    if (x.totals_trace && (s = check_device_ptr(ctx, x.totals_trace, std::string(who) + ": totals_out")))
        return s;
    if (x.totals_final && (s = check_device_ptr(ctx, x.totals_final, std::string(who) + ": totals"))) return s;
    const double *dpersp = persp;
    if (!persp_on_device) {
        for (int32_t i = 0; i < n; ++i) {
            const double *p = persp + 3 * ((size_t)first + (size_t)i * stride);
            if (!finite3(p)) return fail(NBT_ERR_INVALID_ARG, std::string(who) + ": non-finite perspective " +
                                                                   std::to_string(first + i * stride));
            if (p[0] == poi[0] && p[1] == poi[1] && p[2] == poi[2])
                return fail(NBT_ERR_DEGENERATE, std::string(who) + ": perspective " +
                                                    std::to_string(first + i * stride) + " coincides with the PoI");
        }
        if ((s = stage_h2d(ctx, ctx->stage_in[0], ctx->persp, persp, (size_t)n_persp * 24))) return s;
        dpersp = ctx->persp.as<double>();
    }
    IdLaunch L;
    L.d_persp = dpersp;
    L.n_src = n_persp;
    L.first = first;
    L.stride = stride;
    L.n = n;
    for (int k = 0; k < 3; ++k) L.poi[k] = poi[k];
    L.cam = *cam;
    L.range = range;
    L.ray_rank = x.ray_rank;
    L.ray_world = x.ray_world;
    L.d_totals_trace = x.totals_trace;
    L.d_totals_final = x.totals_final;
    L.gather = x.gather;
    L.gather_row0 = x.gather_row0;
    L.peer_totals = x.peer_totals;
    L.d_peer_totals = x.d_peer_totals;
    L.d_record = x.record;
    if (shard) return launch_id(ctx, m, L);
    size_t xyz_b = (size_t)n * 24, gain_b = (size_t)n * 8, cnt_b = (size_t)n * 32;
    if (out->on_device) {
        L.d_xyz_out = out->xyz;
        L.d_gain_out = out->gain;
        L.d_counts_out = out->counts;
        return launch_id(ctx, m, L);
    }
    if ((s = ctx->out_tmp.ensure(xyz_b + gain_b + cnt_b))) return s;
    char *base = ctx->out_tmp.as<char>();
    L.d_xyz_out = reinterpret_cast<double *>(base);
    L.d_gain_out = reinterpret_cast<double *>(base + xyz_b);
    L.d_counts_out = reinterpret_cast<uint64_t *>(base + xyz_b + gain_b);
    if ((s = launch_id(ctx, m, L))) return s;
    size_t total = xyz_b + gain_b + (out->counts ? cnt_b : 0);
    if ((s = ctx->stage_out.acquire(total))) return s;
    NBT_CUDA(cudaMemcpyAsync(ctx->stage_out.p, base, total, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    const char *h = static_cast<const char *>(ctx->stage_out.p);
    memcpy(out->xyz, h, xyz_b);
    memcpy(out->gain, h + xyz_b, gain_b);
    if (out->counts) memcpy(out->counts, h + xyz_b + gain_b, cnt_b);
    return take_device_error(ctx, who);
}

nbt_status nbt_id_compute(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz, int32_t n_persp,
                          int persp_on_device, const nbt_camera *cam, double range, nbt_ig_cloud *out)
{
    return id_common(ctx, m, poi, persp_xyz, n_persp, persp_on_device, 0, 1, cam, range, out, "nbt_id_compute");
}

nbt_status nbt_id_compute_slice(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz,
                                int32_t n_persp, int persp_on_device, int32_t first, int32_t stride,
                                const nbt_camera *cam, double range, nbt_ig_cloud *out)
{
    return id_common(ctx, m, poi, persp_xyz, n_persp, persp_on_device, first, stride, cam, range, out,
                     "nbt_id_compute_slice");
}

nbt_status nbt_id_compute_rays(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz,
                               int32_t n_persp, int persp_on_device, int32_t ray_rank, int32_t ray_world,
                               const nbt_camera *cam, double range, uint64_t *totals_out)
{
    if (ray_world < 1 || ray_rank < 0 || ray_rank >= ray_world || !totals_out)
        return fail(NBT_ERR_INVALID_ARG, "nbt_id_compute_rays: need 0 <= ray_rank < ray_world and totals_out");
    IdExtra x;
    x.ray_rank = ray_rank;
    x.ray_world = ray_world;
    x.totals_trace = totals_out;
    return id_common(ctx, m, poi, persp_xyz, n_persp, persp_on_device, 0, 1, cam, range, nullptr,
                     "nbt_id_compute_rays", x);
}

nbt_status nbt_id_finalize(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz, int32_t n_persp,
                           int persp_on_device, const nbt_camera *cam, double range, const uint64_t *totals,
                           nbt_ig_cloud *out)
{
    if (!totals) return fail(NBT_ERR_INVALID_ARG, "nbt_id_finalize: null totals");
    IdExtra x;
    x.totals_final = totals;
    return id_common(ctx, m, poi, persp_xyz, n_persp, persp_on_device, 0, 1, cam, range, out, "nbt_id_finalize",
                     x);
}

// ------------------------------------------------- peer-memory gather (multi-GPU)

nbt_status nbt_gather_create(nbt_ctx ctx, int32_t rows, int32_t world, int32_t rank, nbt_gather *out)
{
    nbt_status s;
    if (!out) return fail(NBT_ERR_INVALID_ARG, "nbt_gather_create: null out");
    *out = nullptr;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_gather_create during graph capture");
    if (rows < 1 || world < 1 || world > kMaxGatherRanks || rank < 0 || rank >= world)
        return fail(NBT_ERR_INVALID_ARG, "nbt_gather_create: need rows >= 1, 1 <= world <= 16, 0 <= rank < world");
    nbt_gather g = new (std::nothrow) nbt_gather_s();
    if (!g) return fail(NBT_ERR_OUT_OF_MEMORY, "nbt_gather_create");
    cudaError_t e = cudaMalloc(&g->base, (size_t)rows * 64);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_pt, sizeof(PeerTotals));
    if (e == cudaSuccess) {
        // the peer-totals table of nbt_id_compute_rays_gather, kept in device memory (rewritten
        // by every attach) so that a captured ray-split launch copies it device to device
        PeerTotals pt;
        pt.n = world;
        pt.t[rank] = reinterpret_cast<unsigned long long *>(g->base);
        e = cudaMemcpy(g->d_pt, &pt, sizeof pt, cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        if (g->base) cudaFree(g->base);
        if (g->d_pt) cudaFree(g->d_pt);
        delete g;
        return cuda_fail(e, "nbt_gather_create");
    }
    g->ctx = ctx;
    ctx_retain(ctx);
    g->rows = rows;
    g->world = world;
    g->rank = rank;
    g->peer[rank] = g->base;
    *out = g;
    return NBT_OK;
}

nbt_status nbt_gather_export(nbt_gather g, uint8_t handle_out[NBT_PEER_HANDLE_BYTES])
{
    nbt_status s;
    if (!g || !handle_out) return fail(NBT_ERR_INVALID_ARG, "nbt_gather_export: null argument");
    if ((s = bind(g->ctx))) return s;
    static_assert(sizeof(cudaIpcMemHandle_t) <= NBT_PEER_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    NBT_CUDA(cudaIpcGetMemHandle(&h, g->base));
    memset(handle_out, 0, NBT_PEER_HANDLE_BYTES);
    memcpy(handle_out, &h, sizeof h);
    return NBT_OK;
}

nbt_status nbt_gather_attach(nbt_gather g, int32_t peer_rank, const uint8_t handle[NBT_PEER_HANDLE_BYTES])
{
    nbt_status s;
    if (!g || !handle || peer_rank < 0 || peer_rank >= (g ? g->world : 0))
        return fail(NBT_ERR_INVALID_ARG, "nbt_gather_attach: bad argument");
    if (peer_rank == g->rank) return NBT_OK;           // own rows: the local buffer
    if ((s = bind(g->ctx))) return s;
    if (g->peer[peer_rank]) return fail(NBT_ERR_STATE, "nbt_gather_attach: rank already attached");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void *p = nullptr;
    NBT_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    g->peer[peer_rank] = static_cast<char *>(p);
    PeerTotals pt;
    pt.n = g->world;
    for (int r = 0; r < g->world; ++r) pt.t[r] = reinterpret_cast<unsigned long long *>(g->peer[r]);
    NBT_CUDA(cudaMemcpy(g->d_pt, &pt, sizeof pt, cudaMemcpyHostToDevice));
    return NBT_OK;
}

nbt_status nbt_gather_rows(nbt_gather g, nbt_ig_cloud *rows_out)
{
    if (!g || !rows_out) return fail(NBT_ERR_INVALID_ARG, "nbt_gather_rows: null argument");
    rows_out->xyz = reinterpret_cast<double *>(g->base);
    rows_out->gain = reinterpret_cast<double *>(g->base + (size_t)g->rows * 24);
    rows_out->counts = reinterpret_cast<uint64_t *>(g->base + (size_t)g->rows * 32);
    rows_out->on_device = 1;
    return NBT_OK;
}

nbt_status nbt_id_compute_gather(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz,
                                 int32_t n_persp, int persp_on_device, int32_t first, int32_t stride, int32_t row0,
                                 const nbt_camera *cam, double range, nbt_gather g)
{
    if (!g || g->ctx != ctx) return fail(NBT_ERR_STATE, "nbt_id_compute_gather: gather of another ctx");
    if (row0 < 0 || n_persp < 0 || (int64_t)row0 + n_persp > g->rows)
        return fail(NBT_ERR_INVALID_ARG, "nbt_id_compute_gather: need 0 <= row0 and row0 + n_persp <= rows");
    GatherDst dst;
    dst.n = g->world;
    for (int r = 0; r < g->world; ++r) {
        if (!g->peer[r]) return fail(NBT_ERR_STATE, "nbt_id_compute_gather: rank " + std::to_string(r) +
                                                        " not attached");
        dst.xyz[r] = reinterpret_cast<double *>(g->peer[r]);
        dst.gain[r] = reinterpret_cast<double *>(g->peer[r] + (size_t)g->rows * 24);
        dst.counts[r] = reinterpret_cast<unsigned long long *>(g->peer[r] + (size_t)g->rows * 32);
    }
    IdExtra x;
    x.gather = &dst;
    x.gather_row0 = row0;
    return id_common(ctx, m, poi, persp_xyz, n_persp, persp_on_device, first, stride, cam, range, nullptr,
                     "nbt_id_compute_gather", x);
}

nbt_status nbt_gather_zero(nbt_gather g)
{
    nbt_status s;
    if (!g) return fail(NBT_ERR_INVALID_ARG, "nbt_gather_zero: null gather");
    if ((s = bind(g->ctx))) return s;
    NBT_CUDA(cudaMemsetAsync(g->base, 0, (size_t)g->rows * 64, g->ctx->stream));
    return NBT_OK;
}

nbt_status nbt_id_compute_rays_gather(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz,
                                      int32_t n_persp, int persp_on_device, const nbt_camera *cam, double range,
                                      nbt_gather g)
{
    if (!g || g->ctx != ctx) return fail(NBT_ERR_STATE, "nbt_id_compute_rays_gather: gather of another ctx");
    if (n_persp < 0 || (int64_t)n_persp * NBT_ID_TOTALS * 8 > (int64_t)g->rows * 64)
        return fail(NBT_ERR_INVALID_ARG, "nbt_id_compute_rays_gather: the totals do not fit the gather buffers");
    PeerTotals pt;
    pt.n = g->world;
    for (int r = 0; r < g->world; ++r) {
        if (!g->peer[r]) return fail(NBT_ERR_STATE, "nbt_id_compute_rays_gather: rank " + std::to_string(r) +
                                                        " not attached");
        pt.t[r] = reinterpret_cast<unsigned long long *>(g->peer[r]);
    }
    IdExtra x;
    x.ray_rank = g->rank;
    x.ray_world = g->world;
    x.peer_totals = &pt;
    x.d_peer_totals = g->d_pt;
    return id_common(ctx, m, poi, persp_xyz, n_persp, persp_on_device, 0, 1, cam, range, nullptr,
                     "nbt_id_compute_rays_gather", x);
}

void nbt_gather_destroy(nbt_gather g)
{
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    for (int r = 0; r < g->world; ++r)
        if (g->peer[r] && r != g->rank) cudaIpcCloseMemHandle(g->peer[r]);
    if (g->base) cudaFree(g->base);
    if (g->d_pt) cudaFree(g->d_pt);
    nbt_ctx ctx = g->ctx;
    delete g;
    ctx_release(ctx);
}

// ---------------------------------------------------------- ID buffer + IDW

nbt_status nbt_idbuf_create(nbt_ctx ctx, int32_t capacity_nb, int32_t max_persp, nbt_idbuf *out)
{
    nbt_status s;
    if (!out) return fail(NBT_ERR_INVALID_ARG, "nbt_idbuf_create: null out");
    *out = nullptr;
    if ((s = bind(ctx))) return s;
    if (capacity_nb < 1 || capacity_nb > 64 || max_persp < 1)
        return fail(NBT_ERR_INVALID_ARG, "nbt_idbuf_create: need 1 <= capacity <= 64 and max_persp >= 1");
    nbt_idbuf b = new (std::nothrow) nbt_idbuf_s();
    if (!b) return fail(NBT_ERR_OUT_OF_MEMORY, "nbt_idbuf_create");
    b->ctx = ctx;
    ctx_retain(ctx);
    b->capacity = capacity_nb;
    b->max_persp = max_persp;
    cudaError_t e = cudaMalloc(&b->d_xyz, (size_t)capacity_nb * max_persp * 24);
    if (e == cudaSuccess) e = cudaMalloc(&b->d_gain, (size_t)capacity_nb * max_persp * 8);
    if (e == cudaSuccess) e = cudaMalloc(&b->d_meta, 65 * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(b->d_meta, 0, 65 * sizeof(int32_t), ctx->stream);
    if (e != cudaSuccess) {
        nbt_idbuf_destroy(b);
        return cuda_fail(e, "nbt_idbuf_create");
    }
    *out = b;
    return NBT_OK;
}

nbt_status nbt_idbuf_push(nbt_idbuf b, const nbt_ig_cloud *cloud, int32_t n)
{
    if (!b || !cloud) return fail(NBT_ERR_INVALID_ARG, "nbt_idbuf_push: null argument");
    nbt_ctx ctx = b->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (n < 1 || n > b->max_persp) return fail(NBT_ERR_INVALID_ARG, "nbt_idbuf_push: need 1 <= n <= max_persp");
    if (!cloud->xyz || !cloud->gain) return fail(NBT_ERR_INVALID_ARG, "nbt_idbuf_push: null cloud buffers");
    const double *sx = cloud->xyz, *sg = cloud->gain;
    if (!cloud->on_device) {
        if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_idbuf_push: host cloud during graph capture");
        if ((s = ctx->out_tmp.ensure((size_t)n * 32)) || (s = ctx->stage_in[2].acquire((size_t)n * 32))) return s;
        memcpy(ctx->stage_in[2].p, cloud->xyz, (size_t)n * 24);
        memcpy((char *)ctx->stage_in[2].p + (size_t)n * 24, cloud->gain, (size_t)n * 8);
        NBT_CUDA(cudaMemcpyAsync(ctx->out_tmp.p, ctx->stage_in[2].p, (size_t)n * 32, cudaMemcpyHostToDevice,
                                 ctx->stream));
        if ((s = ctx->stage_in[2].mark(ctx->stream))) return s;
        sx = ctx->out_tmp.as<double>();
        sg = sx + 3 * (size_t)n;
    }
    if ((s = launch_idbuf_push(ctx, b, sx, sg, n))) return s;
    if (b->count < b->capacity) b->count++;       // host mirror: only after the push is enqueued
    return NBT_OK;
}

nbt_status nbt_idbuf_clear(nbt_idbuf b)
{
    if (!b) return fail(NBT_ERR_INVALID_ARG, "nbt_idbuf_clear: null buffer");
    nbt_status s;
    if ((s = bind(b->ctx))) return s;
    b->count = 0;
    NBT_CUDA(cudaMemsetAsync(b->d_meta, 0, 65 * sizeof(int32_t), b->ctx->stream));
    return NBT_OK;
}

int32_t nbt_idbuf_size(nbt_idbuf b) { return b ? b->count : 0; }

nbt_status nbt_ig_query(nbt_idbuf b, const double *query_xyz, int32_t n_q, int q_on_device, double power_p,
                        double zero_eps, int32_t normalize_weights, double *g_out, int out_on_device)
{
    return nbt_ig_query_knn(b, query_xyz, n_q, q_on_device, power_p, zero_eps, normalize_weights, 0, g_out,
                            out_on_device);
}

nbt_status nbt_ig_query_knn(nbt_idbuf b, const double *query_xyz, int32_t n_q, int q_on_device, double power_p,
                            double zero_eps, int32_t normalize_weights, int32_t knn, double *g_out, int out_on_device)
{
    if (!b) return fail(NBT_ERR_INVALID_ARG, "nbt_ig_query: null buffer");
    if (knn < 0 || knn > 16) return fail(NBT_ERR_INVALID_ARG, "nbt_ig_query_knn: knn must lie in [0, 16]");
    nbt_ctx ctx = b->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (b->count == 0) return fail(NBT_ERR_EMPTY, "nbt_ig_query: no distribution available");
    if (n_q < 0 || (n_q > 0 && (!query_xyz || !g_out)) || !(power_p >= 0) || !isfinite(power_p) ||
        !(zero_eps >= 0) || !isfinite(zero_eps))
        return fail(NBT_ERR_INVALID_ARG, "nbt_ig_query: bad argument");
    if (n_q == 0) return NBT_OK;
    if (ctx->capturing && (!q_on_device || !out_on_device))
        return fail(NBT_ERR_STATE, "nbt_ig_query: host buffers during graph capture");
    const double *dq = query_xyz;
    if (!q_on_device) {
        for (int32_t i = 0; i < n_q; ++i)
            if (!finite3(query_xyz + 3 * (size_t)i)) return fail(NBT_ERR_INVALID_ARG, "nbt_ig_query: non-finite query");
        if ((s = stage_h2d(ctx, ctx->stage_in[2], ctx->queries, query_xyz, (size_t)n_q * 24))) return s;
        dq = ctx->queries.as<double>();
    }
    double *dout = g_out;
    if (!out_on_device) {
        if ((s = ctx->qout.ensure((size_t)n_q * 8))) return s;
        dout = ctx->qout.as<double>();
    }
    if ((s = launch_idw(ctx, b, dq, n_q, power_p, zero_eps, normalize_weights, dout, knn))) return s;
    if (!out_on_device) return d2h_sync(ctx, g_out, dout, (size_t)n_q * 8);
    return NBT_OK;
}

nbt_status nbt_info_cost(nbt_idbuf b, const double *pose_xyz, const double *pose_axis, int32_t n_traj,
                         int32_t per, int poses_on_device, const double poi[3], double cos_theta_cut, double w_i,
                         double eps, double power_p, double zero_eps, int32_t normalize, double *o_out, double *g_out,
                         double *c_out, int out_on_device)
{
    if (!b) return fail(NBT_ERR_INVALID_ARG, "nbt_info_cost: null buffer");
    nbt_ctx ctx = b->ctx;
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (b->count == 0) return fail(NBT_ERR_EMPTY, "nbt_info_cost: no distribution available");
    if (n_traj < 0 || per < 1 || (n_traj > 0 && (!pose_xyz || !pose_axis || !c_out)) || !poi || !finite3(poi) ||
        !isfinite(cos_theta_cut) || !isfinite(w_i) || !isfinite(eps) || !(power_p >= 0) || !isfinite(power_p) ||
        !(zero_eps >= 0) || (int64_t)n_traj * per > (1ll << 30))
        return fail(NBT_ERR_INVALID_ARG, "nbt_info_cost: bad argument");
    if (n_traj == 0) return NBT_OK;
    const size_t n = (size_t)n_traj * per;
    if (ctx->capturing && (!poses_on_device || !out_on_device))
        return fail(NBT_ERR_STATE, "nbt_info_cost: host buffers during graph capture");
    InfoCostArgs a;
    a.n_traj = n_traj;
    a.per = per;
    for (int k = 0; k < 3; ++k) a.poi[k] = poi[k];
    a.cos_cut = cos_theta_cut;
    a.w_i = w_i;
    a.eps = eps;
    if (poses_on_device) {
        a.pos = pose_xyz;
        a.axis = pose_axis;
    } else {
        for (size_t i = 0; i < n; ++i) {
            const double *p = pose_xyz + 3 * i, *ax = pose_axis + 3 * i;
            if (!finite3(p) || !finite3(ax)) return fail(NBT_ERR_INVALID_ARG, "nbt_info_cost: non-finite pose");
            double d0 = poi[0] - p[0], d1 = poi[1] - p[1], d2 = poi[2] - p[2];
            if (sqrt((d0 * d0 + d1 * d1) + d2 * d2) < 1e-9)
                return fail(NBT_ERR_DEGENERATE, "nbt_info_cost: pose " + std::to_string(i) + " at the PoI");
        }
        if ((s = ctx->poses.ensure(n * 48)) || (s = ctx->stage_in[2].acquire(n * 48))) return s;
        memcpy(ctx->stage_in[2].p, pose_xyz, n * 24);
        memcpy((char *)ctx->stage_in[2].p + n * 24, pose_axis, n * 24);
        NBT_CUDA(cudaMemcpyAsync(ctx->poses.p, ctx->stage_in[2].p, n * 48, cudaMemcpyHostToDevice, ctx->stream));
        if ((s = ctx->stage_in[2].mark(ctx->stream))) return s;
        a.pos = ctx->poses.as<double>();
        a.axis = ctx->poses.as<double>() + 3 * n;
    }
    double *tmp = nullptr;
    if (out_on_device) {
        a.o_out = o_out; a.g_out = g_out; a.c_out = c_out;
    } else {
        if ((s = ctx->qout.ensure(n * 16 + (size_t)n_traj * 8))) return s;
        tmp = ctx->qout.as<double>();
        a.o_out = tmp; a.g_out = tmp + n; a.c_out = tmp + 2 * n;
    }
    if ((s = launch_info_cost(ctx, b, a, power_p, zero_eps, normalize))) return s;
    if (out_on_device) return NBT_OK;
    const size_t total = n * 16 + (size_t)n_traj * 8;
    if ((s = ctx->stage_out.acquire(total))) return s;
    NBT_CUDA(cudaMemcpyAsync(ctx->stage_out.p, tmp, total, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    const double *h = static_cast<const double *>(ctx->stage_out.p);
    if (o_out) memcpy(o_out, h, n * 8);
    if (g_out) memcpy(g_out, h + n, n * 8);
    memcpy(c_out, h + 2 * n, (size_t)n_traj * 8);
    return take_device_error(ctx, "nbt_info_cost");
}

void nbt_idbuf_destroy(nbt_idbuf b)
{
    if (!b) return;
    cudaSetDevice(b->ctx->device);
    cudaStreamSynchronize(b->ctx->stream);
    if (b->d_xyz) cudaFree(b->d_xyz);
    if (b->d_gain) cudaFree(b->d_gain);
    if (b->d_meta) cudaFree(b->d_meta);
    nbt_ctx ctx = b->ctx;
    delete b;
    ctx_release(ctx);
}

// -------------------------------------------------------------- test hooks

nbt_status nbt_debug_trace(nbt_ctx ctx, nbt_map m, const int32_t *o_q16, const int32_t *e_q16, int32_t n_rays,
                           int32_t max_visits, int32_t *ijk_out, uint8_t *code_out, int32_t *len_out,
                           uint32_t *counts_out)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (!m || m->ctx != ctx) return fail(NBT_ERR_STATE, "nbt_debug_trace: map of another ctx");
    if (n_rays < 0 || max_visits < 1 || (n_rays > 0 && (!o_q16 || !e_q16 || !ijk_out || !code_out || !len_out ||
                                                        !counts_out)))
        return fail(NBT_ERR_INVALID_ARG, "nbt_debug_trace: bad argument");
    if (n_rays == 0) return NBT_OK;
    for (int32_t i = 0; i < 3 * n_rays; ++i)
        if (o_q16[i] <= -(1 << 30) || o_q16[i] >= (1 << 30) || e_q16[i] <= -(1 << 30) || e_q16[i] >= (1 << 30))
            return fail(NBT_ERR_INVALID_ARG, "nbt_debug_trace: coordinate outside (-2^30, 2^30)");
    size_t nr = n_rays, mv = max_visits;
    size_t b_in = nr * 12, b_ijk = nr * mv * 12, b_code = nr * mv, b_len = nr * 4, b_cnt = nr * 16;
    size_t total = 2 * b_in + b_ijk + b_code + b_len + b_cnt + 64;
    if ((s = ctx->dbg.ensure(total))) return s;
    char *base = ctx->dbg.as<char>();
    int32_t *d_o = (int32_t *)base, *d_e = (int32_t *)(base + b_in);
    int32_t *d_ijk = (int32_t *)(base + 2 * b_in);
    int32_t *d_len = (int32_t *)(base + 2 * b_in + b_ijk);
    uint32_t *d_cnt = (uint32_t *)(base + 2 * b_in + b_ijk + b_len);
    uint8_t *d_code = (uint8_t *)(base + 2 * b_in + b_ijk + b_len + b_cnt);
    NBT_CUDA(cudaMemcpyAsync(d_o, o_q16, b_in, cudaMemcpyHostToDevice, ctx->stream));
    NBT_CUDA(cudaMemcpyAsync(d_e, e_q16, b_in, cudaMemcpyHostToDevice, ctx->stream));
    const bool need_wide = debug_needs_wide(o_q16, e_q16, n_rays);
    if (ctx->opt.walk_width == 32 && need_wide)
        return fail(NBT_ERR_INVALID_ARG, "nbt_debug_trace: int32 walk forced on a segment with |E - O| >= 2^30 - 1");
    const bool wide = ctx->opt.walk_width == 64 || (ctx->opt.walk_width == 0 && need_wide);
    if ((s = launch_debug_trace(ctx, m, d_o, d_e, n_rays, max_visits, d_ijk, d_code, d_len, d_cnt, wide))) return s;
    NBT_CUDA(cudaMemcpyAsync(ijk_out, d_ijk, b_ijk, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaMemcpyAsync(code_out, d_code, b_code, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaMemcpyAsync(len_out, d_len, b_len, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaMemcpyAsync(counts_out, d_cnt, b_cnt, cudaMemcpyDeviceToHost, ctx->stream));
    NBT_CUDA(cudaStreamSynchronize(ctx->stream));
    return NBT_OK;
}

// Per-ray counts of the production trace kernel (its REC instance: the same code, recording
// every closed ray), for per-ray parity against the oracle's perspective_rays.
nbt_status nbt_debug_id_rays(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz, int32_t n,
                             const nbt_camera *cam, double range, uint32_t *ray_counts_out)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (ctx->capturing) return fail(NBT_ERR_STATE, "nbt_debug_id_rays: not inside a graph capture");
    if ((s = check_camera(cam))) return s;
    if (n < 0 || (n > 0 && (!persp_xyz || !ray_counts_out)))
        return fail(NBT_ERR_INVALID_ARG, "nbt_debug_id_rays: bad argument");
    if (n == 0) return NBT_OK;
    const size_t ne = (size_t)cam->width * cam->height + (cam->add_corners ? 4 : 0);
    const size_t bytes = (size_t)n * ne * 5 * sizeof(uint32_t);
    if ((s = ctx->dbg.ensure(bytes))) return s;
    NBT_CUDA(cudaMemsetAsync(ctx->dbg.p, 0xFF, bytes, ctx->stream));     // unwritten rays read as ~0
    std::vector<double> xyz((size_t)n * 3), gain((size_t)n);
    nbt_ig_cloud out{xyz.data(), gain.data(), nullptr, 0};
    IdExtra x;
    x.record = ctx->dbg.as<uint32_t>();
    if ((s = id_common(ctx, m, poi, persp_xyz, n, 0, 0, 1, cam, range, &out, "nbt_debug_id_rays", x))) return s;
    return d2h_sync(ctx, ray_counts_out, ctx->dbg.p, bytes);
}

nbt_status nbt_debug_frames(nbt_ctx ctx, nbt_map m, const double poi[3], const double *persp_xyz, int32_t n,
                            const nbt_camera *cam, double range, int32_t *q16_out, int32_t *status_out)
{
    nbt_status s;
    if ((s = bind(ctx))) return s;
    if (!m || !poi || n < 0 || (n > 0 && (!persp_xyz || !q16_out || !status_out)))
        return fail(NBT_ERR_INVALID_ARG, "nbt_debug_frames: bad argument");
    if ((s = check_camera(cam))) return s;
    if (n == 0) return NBT_OK;
    size_t b_in = (size_t)n * 24, b_out = (size_t)n * 19 * 4;
    if ((s = ctx->dbg.ensure(b_in + b_out + 64))) return s;
    double *d_p = ctx->dbg.as<double>();
    int32_t *d_f = (int32_t *)(ctx->dbg.as<char>() + b_in);
    NBT_CUDA(cudaMemcpyAsync(d_p, persp_xyz, b_in, cudaMemcpyHostToDevice, ctx->stream));
    if ((s = launch_debug_frames(ctx, m, poi, d_p, n, *cam, range, d_f))) return s;
    int32_t *h = new (std::nothrow) int32_t[(size_t)n * 19];
    if (!h) return fail(NBT_ERR_OUT_OF_MEMORY, "nbt_debug_frames");
    cudaError_t e = cudaMemcpyAsync(h, d_f, b_out, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e == cudaSuccess) {
        for (int32_t i = 0; i < n; ++i) {
            memcpy(q16_out + 18 * (size_t)i, h + 19 * (size_t)i, 18 * 4);
            status_out[i] = h[19 * (size_t)i + 18];
        }
    }
    delete[] h;
    if (e != cudaSuccess) return cuda_fail(e, "nbt_debug_frames");
    return NBT_OK;
}

}  // extern "C"
