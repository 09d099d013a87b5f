// The online local Information Distribution on the device.
//
//   k_persp_frames  per perspective: view frame (Q4) and its Q16 quantisation
//                   (Q19), bound checks; zeroes the per-perspective totals.
//   k_id_trace      persistent warps walking 8x4 pixel tiles in lockstep: a warp takes
//                   chunks of one perspective's ray slots from a global counter (handed
//                   out position-major, the image's middle tile rows last), prepares a
//                   tile's 32 rays at once (frame, endpoint on the far plane in registers,
//                   P:158-169, Q27, on the frame's Q16 lattice; DDA init; grid entry) and
//                   walks them together until all have ended (NBT_OPT_TRACE_REFILL_MIN
//                   < 32: per-lane refills from the prepared-ray queue instead).  Each
//                   lane walks the exact integer 3D-DDA (Q13) through the map in batches
//                   of K = 16 voxels: the DDA does not depend on the map, so a batch
//                   computes K voxel indices, issues K independent loads, packs the
//                   codes into one word (visit 0 at the top) and finds the first
//                   Occupied / outside voxel with one clz (early stop) and the
//                   Free count with one popc.  Per-state visit
//                   counts (Eq. 2 as integers, Q26) accumulate in registers and are
//                   flushed warp-combined (one u64 atomic per counter per warp and
//                   perspective) when lanes move to another perspective.  A separate
//                   SHARD instance walks one ray shard (nbt_id_compute_rays).
//   k_id_finalize   g_P = ((T_U g_U + T_F g_F) + T_O g_O) / N_E  (Q26)
//   k_id_finalize_gather  the same rows stored into every rank's peer-mapped buffer
//                   (the all-gather fused into the finalize, nbt_id_compute_gather)
//
// Exact decision with 32-bit arithmetic.  With D = E - O and
// N_a the distance from O to the next boundary along a (Q16 units, S = 65536), the next
// boundary crossed is the axis minimising N_a/|D_a|, ties broken by (positive direction
// first, then x<y<z).  The pairwise terms e_ab = N_a|D_b| - N_b|D_a|, minus a 0/1 tie
// bias, decide "a before b" by their sign.  Every later change of e_ab is a multiple
// of S (a step along a adds S|D_b|), so with e_ab - bias = S q_ab + r (0 <= r < S) the
// sign of q_ab equals the sign of e_ab - bias and q_ab changes by |D_b| (or -|D_a|).
// q_ab is computed once per ray in 64-bit and then kept in int32.  Bound (tight): N_a is
// in [0, S], so q_ab starts in [-|D_a| - 1, |D_b|]; an a-step (taken only while q_ab < 0)
// adds |D_b|, a b-step (only while q_ab >= 0) subtracts |D_a|, a c-step leaves it, so
// q_ab -- and every intermediate value, speculative steps past the ray end included --
// stays in [-|D_a| - 1, |D_b|].  int32 is therefore exact while max |D| < 2^30 - 1, i.e.
// for rays shorter than 16383 voxels per axis; the host picks the 64-bit instance of the
// same code above kInt32MaxVoxels (tests/test_gpu_parity.py::test_int32_bound_*).
#include <stdio.h>

#include <type_traits>

#include "nbt_internal.cuh"
#include "dda.cuh"

namespace nbt {
namespace {
using namespace dda;

constexpr int kFrameInts = 20;   // O, A, Rh, Uh, Rc, Uc (3 each, Q16), status, pad
constexpr int kTotals = 5;       // per perspective: T_U, T_F, T_O, L, T_G (Eq. 2 gain, 1/63 units)
static_assert(kTotals == NBT_ID_TOTALS, "totals layout of nbt_id_compute_rays");
#ifndef NBT_WARPS_PER_BLOCK
#define NBT_WARPS_PER_BLOCK 8
#endif
constexpr int kWarpsPerBlock = NBT_WARPS_PER_BLOCK;
// Trace kernel shape: K voxels per speculative batch; PIPE = in-place software pipeline
// (batch_cycle: the next batch's loads replace the current one's slot by slot, look-ahead
// 2K, so build with NBT_BORDER >= 2K).  K = 16 without pipelining measured best: the
// pipelined shapes spill at the 64-register budget or lose to the doubled speculation
// past a stop (profiles/r01_trace_variants.md); they stay compilable for experiments.
#ifndef NBT_BATCH_K
#define NBT_BATCH_K 16
#endif
#ifndef NBT_PIPE
#define NBT_PIPE false
#endif
constexpr int kBatchK = NBT_BATCH_K;
constexpr bool kPipe = NBT_PIPE;
constexpr int kInt32MaxVoxels = 16000;   // |D_a| bound (voxels) for the int32 decision terms (< 16383)
// Largest chunk of ray slots per work grab (8 tiles): with tile lockstep a warp's last chunk is the
// end-of-launch tail, and 256-slot chunks cut D by 4.7% and C' by 0.7% against 1024 (128: D -5.1%,
// C' -0.2%; 64: D -4.7%, C' +0.6%; profiles/r02_s3_cmax*.log).
// Chunk size = the launch's slots / (32 x resident warps), 64..256 slots: full-size D and C' (>= 8 k
// slots per warp) keep 256, config B keeps 64, and the mid-size launches of one rank's strided shard
// of D get finer chunks for a shorter tail -- 1024 perspectives (N = 4) -2.9%, 512 (N = 8) -4.2%
// against 4 chunks per warp (profiles/r02_s3_shards.log).
#ifndef NBT_CHUNKS_PER_WARP
#define NBT_CHUNKS_PER_WARP 32
#endif
// Chunk order: 1 = position-major, the image's top and bottom rows of tiles first and its middle
// rows last (chunk index c -> perspective c mod n, position c / n taken 0, last, 1, last - 1, ...):
// the middle rows look at the object and stop early, so the launch ends on short tiles -- B -4.8%,
// one rank's D shard at N = 8 -4.4%, D -0.7%, C' -0.2% (profiles/r02_s3_chunk_order.log);
// 0 = perspective-major (round 2).
#ifndef NBT_SPLIT_TAIL
#define NBT_SPLIT_TAIL 2           // chunks per resident warp handed out as halves at the launch's end
#endif
#ifndef NBT_CHUNK_ORDER
#define NBT_CHUNK_ORDER 1
#endif
#ifndef NBT_CHUNK_MAX
#define NBT_CHUNK_MAX 256
#endif
#ifndef NBT_TILE_W
#define NBT_TILE_W 8
#endif
constexpr int kTileW = NBT_TILE_W;       // a warp's 32 rays: a kTileW x kTileH pixel tile
constexpr int kTileH = 32 / kTileW;

// Store kinds (the VB template parameter): kStore2 = 2-bit codes, 16 per word (rows a1, a6);
// kStoreByte = one byte per voxel holding the code alone; kStoreProb = one byte per voxel,
// code in bits 0-1 and the Eq. 2 gain in bits 2-7 (f1).  Byte stores load the voxel's own
// byte, so a visit needs no rotate and the code packs with one shift-add.
constexpr int kStore2 = 2, kStoreByte = 1, kStoreProb = 8;

// Scale of the walk's linear index: the 2-bit linear store walks the code's bit offset 2i
// (its word is ib >> 5 and one left rotate by ib brings the code to bits 30-31, map_store.cuh),
// so a visit needs no separate rotate amount; byte stores walk the byte index i.
template <int L, int VB>
__device__ __forceinline__ constexpr int idx_shift()
{
    return (L == kLayoutLinear && VB == kStore2) ? 1 : 0;
}

// Origin outside the grid (rare): step with explicit bounds checks until the walk
// enters the grid or ends.  Returns true if the ray is finished.
template <typename T, int L, bool RECORD, int SH = 0>
__device__ bool walk_enter(Walk<T> &w, const MapView &m, int32_t *rec_ijk, uint8_t *rec_code, int max_visits)
{
    while (!inside(m, w.vx, w.vy, w.vz)) {
        if (RECORD && w.s < max_visits) {
            rec_ijk[3 * w.s] = w.vx; rec_ijk[3 * w.s + 1] = w.vy; rec_ijk[3 * w.s + 2] = w.vz;
            rec_code[w.s] = 255;
        }
        w.pre++;
        if (w.s == w.n) return true;
        walk_step<T, L, true>(w, m);
        w.s++;
    }
    w.s0 = w.s;
    if (L == kLayoutMorton) {
        const uint32_t dx = dilate3((uint32_t)w.vx), dy = dilate3((uint32_t)w.vy) << 1,
                       dz = dilate3((uint32_t)w.vz) << 2;
        w.xinv = (w.sx > 0 ? m.mx : 0u) | (w.sy > 0 ? m.my : 0u) | (w.sz > 0 ? m.mz : 0u);
        w.rx = (dx ^ w.xinv) & m.mx;
        w.ry = (dy ^ w.xinv) & m.my;
        w.rz = (dz ^ w.xinv) & m.mz;
        w.idx = dx | dy | dz;
    } else {
        w.idx = grid_index<L>(m, w.vx, w.vy, w.vz) << SH;
        w.dX = w.sx * (1 << SH);
        w.dY = w.sy * m.px * (1 << SH);
        w.ndZ = -w.sz * m.pxy * (1 << SH);
    }
    return false;
}

// Per-lane integer accumulators of one perspective: visits per state, in-grid lookups,
// and (8-bit store) the Eq. 2 gain in units of 1/63.
struct Counts { uint32_t u, f, o, l, g; };

// Close a ray that stopped at step s_stop on `code` (2 = Occupied, 3 = left the grid;
// Q14 tail rule: the remaining n - s + 1 visits are all outside, hence Unknown).  ng = the
// in-grid gain (1/63 units) up to and including the stop.
template <typename T>
__device__ __forceinline__ void walk_close_stop(const Walk<T> &w, int policy, uint32_t code, int s_stop, uint32_t nf,
                                                uint32_t ng, Counts &c)
{
    uint32_t l;
    uint32_t u_out = (policy == NBT_OUTSIDE_UNKNOWN) ? w.pre : 0u;
    if (code == 2u) {
        l = (uint32_t)(s_stop - w.s0 + 1);
        c.o += 1;
        c.u += l - nf - 1 + u_out;
    } else {
        l = (uint32_t)(s_stop - w.s0);
        if (policy == NBT_OUTSIDE_UNKNOWN) u_out += (uint32_t)(w.n - s_stop + 1);
        c.u += l - nf + u_out;
    }
    c.f += nf;
    c.l += l;
    c.g += ng + 63u * u_out;
}

template <typename T>
__device__ __forceinline__ void walk_close_end(const Walk<T> &w, int policy, uint32_t nf, uint32_t ng, Counts &c)
{
    const uint32_t l = (uint32_t)(w.n - w.s0 + 1);
    const uint32_t u_out = (policy == NBT_OUTSIDE_UNKNOWN) ? w.pre : 0u;
    c.u += l - nf + u_out;
    c.f += nf;
    c.l += l;
    c.g += ng + 63u * u_out;
}

// A batch of K visits: the loaded map words and, per visit (2-bit store), the code's bit
// offset, the left rotate that brings the code to bits 30-31.
template <int K>
struct Batch {
    uint32_t wd[K];
    uint32_t rot[K];
};

// Packed codes of a batch: visit k at bits 31-2k..30-2k (visit 0 at the top).
template <int K>
__device__ __forceinline__ constexpr uint32_t batch_mask()
{
    return K >= 16 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> (2 * K));
}

#ifndef NBT_MAP_LOAD
#define NBT_MAP_LOAD 0
#endif
// Map word load of the walk: 0 = ld.global.nc (default), 1 = L1::evict_last, 2 = L1::evict_first,
// 3 = L1::no_allocate (experiments).
__device__ __forceinline__ uint32_t load_map_word(const uint32_t *p)
{
#if NBT_MAP_LOAD == 1
    uint32_t v;
    asm("ld.global.nc.L1::evict_last.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#elif NBT_MAP_LOAD == 2
    uint32_t v;
    asm("ld.global.nc.L1::evict_first.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#elif NBT_MAP_LOAD == 3
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

// Step table (NBT_DDA_TABLE experiment, linear layout, int32 terms): per lane, the three
// possible updates (dq_xy, dq_xz, dq_yz, d_idx) of a step along x, y, z in shared memory,
// written when the lane takes a ray; a step is then the axis choice (2 LOP3 + 2 SHF), one
// 16-byte shared load and 4 adds instead of the 9 flag multiply-adds of the round-2 walk_step
// (walk_step itself is now 4 compares and 9 predicated adds, dda.cuh).
#ifndef NBT_DDA_TABLE
#define NBT_DDA_TABLE 0
#endif
constexpr bool kDdaTable = NBT_DDA_TABLE != 0;

// Shared-window address of the lane's z-step entry (the x and y entries sit 1024 and 512
// bytes below it).  The table accesses are volatile asm so that the compiler keeps the
// lane's stores before its loads.
__device__ __forceinline__ void table_put_row(uint32_t a, int x, int y, int z, int w)
{
    asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}

template <typename T>
__device__ __forceinline__ void table_put(uint32_t tz, const Walk<T> &w)
{
    table_put_row(tz - 1024u, (int)w.ay, (int)w.az, 0, w.dX);          // x step
    table_put_row(tz - 512u, (int)-w.ax, 0, (int)w.az, w.dY);          // y step
    table_put_row(tz, 0, (int)-w.ax, (int)-w.ay, -w.ndZ);              // z step
}

template <typename T>
__device__ __forceinline__ void walk_step_table(Walk<T> &w, uint32_t tz)
{
    const int t1 = w.qxy & w.qxz;                // sign: x first
    const int t2 = w.qyz & ~t1;                  // sign: y first
    const int px = (int)((unsigned)t1 >> 31);
    const int py = (int)((unsigned)t2 >> 31);
    const uint32_t a = (uint32_t)mad_i32(px, -1024, mad_i32(py, -512, (int)tz));   // axis 2 - 2 px - py
    int dx, dy, dz, di;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(dx), "=r"(dy), "=r"(dz), "=r"(di) : "r"(a));
    w.qxy = mad_i32(1, dx, w.qxy);               // the adds as IMADs: the FMA pipe has room, the ALU not
    w.qxz = mad_i32(1, dy, w.qxz);
    w.qyz = mad_i32(1, dz, w.qyz);
    w.idx = (uint32_t)mad_i32(1, di, (int)w.idx);
}

#ifndef NBT_BYTE_ASM
#define NBT_BYTE_ASM 1
#endif
#ifndef NBT_ADDR_LEA
#define NBT_ADDR_LEA 1     // 0: the 2-bit word address by SHF + IMAD.WIDE (A/B builds)
#endif
// Issue the K loads of the next K visits (the DDA does not depend on the map, so
// this runs ahead of the codes) and advance the DDA by K steps.
template <typename T, int L, int VB, int K, bool TAB = false>
__device__ __forceinline__ void batch_issue(Walk<T> &w, const MapView &m, Batch<K> &b, uint32_t tz = 0)
{
    const uint8_t *bytes = reinterpret_cast<const uint8_t *>(m.words);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (VB == kStore2) {
            const uint32_t ib = L == kLayoutLinear ? w.idx : (w.idx << 1);   // the code's bit offset
            b.rot[k] = ib;                       // rotate amounts are taken mod 32
#if NBT_ADDR_LEA
            // the word address by a 64-bit shift and add: ptxas emits SHF + LEA + LEA.HI.X (ALU
            // pipe) instead of SHF + IMAD.WIDE (FMA pipe, which the predicated step already fills)
            const uint32_t *a;
            asm("{\n\t.reg .u64 t;\n\tcvt.u64.u32 t, %1;\n\tshr.u64 t, t, 5;\n\tshl.b64 t, t, 2;\n\t"
                "add.s64 %0, %2, t;\n\t}" : "=l"(a) : "r"(ib), "l"(m.words));
            b.wd[k] = load_map_word(a);
#else
            b.wd[k] = load_map_word(m.words + (ib >> 5));
#endif
        } else if (NBT_BYTE_ASM) {
            // the byte lands zero-extended in a 32-bit register: the packing shift-adds need
            // no mask (through __ldg the compiler re-masks every byte before packing)
            asm("ld.global.nc.u8 %0, [%1];" : "=r"(b.wd[k]) : "l"(bytes + w.idx));
        } else {
            b.wd[k] = __ldg(bytes + w.idx);
        }
        if constexpr (TAB)
            walk_step_table(w, tz);
        else
            walk_step<T, L, false, VB == kStore2>(w, m);
    }
}

// Append the code of visit k of a batch below the codes packed so far: 2-bit store, one
// rotate (code to bits 30-31) and one funnel shift; byte stores, one shift-add.
#ifndef NBT_BYTE_REV
#define NBT_BYTE_REV 0
#endif
// NBT_BYTE_REV = 1 (experiment): the byte store's batch word packed bottom-up (visit k at bits
// 2k+1..2k), each code entering at the top by one funnel shift right -- an ALU instruction where
// the top-down shift-add is an FMA-pipe IMAD; C' +0.5% (profiles/r02_s4_revpack.log), not the default.
template <int VB>
constexpr bool rev_pack() { return VB == kStoreByte && NBT_BYTE_REV; }

template <int VB, int K>
__device__ __forceinline__ uint32_t batch_push(uint32_t bits, const Batch<K> &b, int k)
{
    if (VB == kStore2) return __funnelshift_l(__funnelshift_l(b.wd[k], b.wd[k], b.rot[k]), bits, 2);
    if (rev_pack<VB>()) return __funnelshift_r(bits, b.wd[k], 2);  // (bits >> 2) | code << 30
    if (VB == kStoreByte) return bits * 4u + b.wd[k];             // the byte is the code (< 4)
    return (bits << 2) | (b.wd[k] & 3u);
}

// The packed codes of a whole batch, visit k at bits 31-2k..30-2k (bottom-up stores: 2k+1..2k).
template <int VB, int K>
__device__ __forceinline__ uint32_t batch_bits(const Batch<K> &b)
{
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) bits = batch_push<VB, K>(bits, b, k);
    if (rev_pack<VB>()) return K >= 16 ? bits : bits >> (32 - 2 * K);
    return K >= 16 ? bits : bits << (32 - 2 * K);
}

// Close or advance the walk after the batch holding visits s..s+K-1, whose codes are
// packed in `bits` (visit k at bits 31-2k..30-2k; with the 8-bit store, whose gains sum to
// gsum / are read from b).  Returns true when the ray is finished (counts added to c): first
// code >= 2 by one clz (Occupied: early stop; 3: left the grid), Free voxels by one popc.
template <typename T, int VB, int K>
__device__ __forceinline__ bool batch_finish(Walk<T> &w, uint32_t bits, uint32_t gsum, const Batch<K> &b,
                                             int policy, Counts &c)
{
    constexpr bool REV = rev_pack<VB>();        // visit k at bits 2k+1..2k
    const int left = w.n - w.s + 1;             // visits remaining, including the current one
    const uint32_t valid = REV ? (left >= K ? (K >= 16 ? 0xFFFFFFFFu : (1u << (2 * K)) - 1u)
                                            : 0xFFFFFFFFu >> (32 - 2 * left))
                               : (left >= K ? batch_mask<K>() : ~(0xFFFFFFFFu >> (2 * left)));   // 1 <= left < 16
    const uint32_t stop = bits & valid & 0xAAAAAAAAu;   // codes 2 (Occupied) and 3 (outside)
    if (stop || left <= K) {
        // last batch of the ray: only visits up to the stop (or the end) count.  The same counts
        // as walk_close_stop / walk_close_end in branch-free form: visit `last` is the stop (code
        // 2 Occupied: counted; 3: left the grid, Q14) or the ray's end (code 0 or 1).
        const int last = stop ? (REV ? (__ffs(stop) - 1) >> 1 : __clz(stop) >> 1) : left - 1;
        const uint32_t upto = REV ? 0xFFFFFFFFu >> (30 - 2 * last)              // visits 0..last
                                  : ~((0xFFFFFFFFu >> (2 * last)) >> 2);
        const uint32_t code = REV ? (bits >> (2 * last)) & 3u : (bits << (2 * last)) >> 30;
        const uint32_t nf = w.nf + __popc(bits & ~(bits >> 1) & upto & 0x55555555u);   // codes 01 only
        const uint32_t o = code == 2u, out = code == 3u;
        const uint32_t l = (uint32_t)(w.s - w.s0 + last + 1) - out;      // in-grid lookups
        uint32_t u_out = 0;                                              // Unknown visits outside (Q14)
        if (policy == NBT_OUTSIDE_UNKNOWN) u_out = w.pre + out * (uint32_t)(w.n - w.s - last + 1);
        c.o += o;
        c.f += nf;
        c.l += l;
        c.u += l - nf - o + u_out;
        if (VB == kStoreProb) {
            uint32_t ng = w.ng;
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (k <= last) ng += b.wd[k] >> 2;
            c.g += ng + 63u * u_out;
        }
        return true;
    }
    w.nf += __popc(bits & 0x55555555u);
    if (VB == kStoreProb) w.ng += gsum;
    w.s += K;
    return false;
}

// Consume the batch holding visits s..s+K-1 (see batch_finish).
template <typename T, int VB, int K>
__device__ __forceinline__ bool batch_consume(Walk<T> &w, const Batch<K> &b, int policy, Counts &c)
{
    uint32_t gsum = 0;
    if (VB == kStoreProb) {
#pragma unroll
        for (int k = 0; k < K; ++k) gsum += b.wd[k] >> 2;      // Eq. 2 gain in 1/63 units
    }
    return batch_finish<T, VB, K>(w, batch_bits<VB, K>(b), gsum, b, policy, c);
}

// In-place software pipeline (stores without a gain): extract the codes of the batch in b
// (visits s..s+K-1) and, slot by slot, overwrite it with the loads of the next K visits, so
// every load has a whole batch of DDA work to arrive before it is read.  Look-ahead 2K
// voxels past the consumed position (kBorder >= 2K).
template <typename T, int L, int VB, int K>
__device__ __forceinline__ uint32_t batch_cycle(Walk<T> &w, const MapView &m, Batch<K> &b)
{
    const uint8_t *bytes = reinterpret_cast<const uint8_t *>(m.words);
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        bits = batch_push<VB, K>(bits, b, k);
        if (VB == kStore2) {
            const uint32_t ib = L == kLayoutLinear ? w.idx : (w.idx << 1);
            b.rot[k] = ib;
            b.wd[k] = __ldg(m.words + (ib >> 5));
        } else {
            b.wd[k] = __ldg(bytes + w.idx);
        }
        walk_step<T, L, false, VB == kStore2>(w, m);
    }
    return K >= 16 ? bits : bits << (32 - 2 * K);
}

// ------------------------------------------------------------------ frames (a4)

__device__ __forceinline__ bool rne_q16(double v, int *out)
{
    double q = __dmul_rn(v, 65536.0);
    if (!(fabs(q) < 1073741824.0)) return false;
    *out = __double2int_rn(q);   // round half to even
    return true;
}

__device__ __forceinline__ double dot3_sq(double a, double b, double c)
{
    return __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c));
}

struct FrameArgs {
    const double *persp;
    int32_t first, stride, n;
    double poi[3];
    double origin[3];
    double voxel_size;
    double range;
    nbt_camera cam;
};

// Frame of perspective p: fwd = unit(PoI - p), right = unit(fwd x z) or
// unit(fwd x x) when |fwd x z| < 1e-6 (Q4), up = right x fwd; every product, sum
// and quotient rounded once (no FMA contraction) so the result is reproducible.
__device__ int make_frame(const FrameArgs &A, const double p[3], int f[18])
{
    double d0 = __dsub_rn(A.poi[0], p[0]), d1 = __dsub_rn(A.poi[1], p[1]), d2 = __dsub_rn(A.poi[2], p[2]);
    if (d0 == 0.0 && d1 == 0.0 && d2 == 0.0) return NBT_ERR_DEGENERATE;
    if (!(isfinite(d0) && isfinite(d1) && isfinite(d2))) return NBT_ERR_INVALID_ARG;
    double nrm = __dsqrt_rn(dot3_sq(d0, d1, d2));
    double fw[3] = {__ddiv_rn(d0, nrm), __ddiv_rn(d1, nrm), __ddiv_rn(d2, nrm)};
    double c[3] = {fw[1], -fw[0], 0.0};
    double nc = __dsqrt_rn(dot3_sq(c[0], c[1], c[2]));
    if (nc < 1e-6) {
        c[0] = 0.0; c[1] = fw[2]; c[2] = -fw[1];
        nc = __dsqrt_rn(dot3_sq(c[0], c[1], c[2]));
    }
    double rt[3] = {__ddiv_rn(c[0], nc), __ddiv_rn(c[1], nc), __ddiv_rn(c[2], nc)};
    double up[3] = {__dsub_rn(__dmul_rn(rt[1], fw[2]), __dmul_rn(rt[2], fw[1])),
                    __dsub_rn(__dmul_rn(rt[2], fw[0]), __dmul_rn(rt[0], fw[2])),
                    __dsub_rn(__dmul_rn(rt[0], fw[1]), __dmul_rn(rt[1], fw[0]))};
    double s = A.voxel_size;
    double rs = __ddiv_rn(A.range, s);
    double hx = __ddiv_rn(rs, __dmul_rn(2.0, A.cam.fx));
    double hy = __ddiv_rn(rs, __dmul_rn(2.0, A.cam.fy));
    double ch = __dmul_rn(rs, A.cam.tan_half_fov_h);
    double cv = __dmul_rn(rs, A.cam.tan_half_fov_v);
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        ok &= rne_q16(__ddiv_rn(__dsub_rn(p[k], A.origin[k]), s), &f[k]);
        ok &= rne_q16(__dmul_rn(rs, fw[k]), &f[3 + k]);
        ok &= rne_q16(__dmul_rn(hx, rt[k]), &f[6 + k]);
        ok &= rne_q16(__dmul_rn(hy, up[k]), &f[9 + k]);
        ok &= rne_q16(__dmul_rn(ch, rt[k]), &f[12 + k]);
        ok &= rne_q16(__dmul_rn(cv, up[k]), &f[15 + k]);
    }
    if (!ok) return NBT_ERR_INVALID_ARG;
    // every ray endpoint must stay inside (-2^30, 2^30): E is affine in the lattice
    // offsets, so checking the four lattice corners (and the corner rays) suffices.
    const long long lim = 1073741824LL;
    long long mw = A.cam.width - 1, mh = A.cam.height - 1;
    for (int q = 0; q < 8; ++q) {
        if (q >= 4 && !A.cam.add_corners) break;
        long long sr = (q & 1) ? 1 : -1, su = (q & 2) ? 1 : -1;
        for (int k = 0; k < 3; ++k) {
            long long e = (long long)f[k] + f[3 + k];
            e += (q < 4) ? sr * mw * f[6 + k] + su * mh * f[9 + k] : sr * f[12 + k] + su * f[15 + k];
            if (e <= -lim || e >= lim) return NBT_ERR_INVALID_ARG;
        }
    }
    return NBT_OK;
}

__global__ void k_persp_frames(FrameArgs A, int32_t *__restrict__ frames, unsigned long long *__restrict__ totals,
                               int *work_counter, int *err)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *work_counter = 0;
    if (i >= A.n) return;
    const double *pp = A.persp + 3 * (size_t)(A.first + (size_t)i * A.stride);
    double p[3] = {pp[0], pp[1], pp[2]};
    int f[18] = {0};
    int st = make_frame(A, p, f);
    int32_t *dst = frames + (size_t)i * kFrameInts;
#pragma unroll
    for (int k = 0; k < 18; ++k) dst[k] = st ? 0 : f[k];
    dst[18] = st;
    dst[19] = 0;
#pragma unroll
    for (int k = 0; k < kTotals; ++k) totals[kTotals * (size_t)i + k] = 0ull;
    if (st) atomicCAS(err, 0, st);
}

// ------------------------------------------------------------ trace (a5-a8)

struct TraceArgs {
    MapView m;
    const int32_t *__restrict__ frames;
    unsigned long long *totals;
    int *work_counter;
    int W, H, add_corners;
    int tiled;                  // 1: warp-coherent 8x4 pixel tiles
    int Wt;                     // tiles per row
    int n_tile_slots;           // tiles * 32 (tiled) or W*H
    int slots;                  // slots per perspective (incl. 4 corner slots on ray rank 0)
    int chunk;                  // slots per chunk (multiple of 32)
    int chunks_per_persp;
    int total_chunks;
    int min_refill;             // idle lanes needed before a warp refills (experiments)
    int ray_rank, ray_world;    // ray shard: this call walks 32-slot units u = ray_rank mod ray_world
    int local_tile_slots;       // lattice slots of this shard (its units * 32)
    int split_from;             // chunks from this index on are handed out as two half chunks
    int total_grabs;            // split_from + 2 * (total_chunks - split_from)
};

// SHARD instance: the peer totals of a fused ray split live in the work-counter buffer, after
// the counter (n = 0: add into the call's totals).  Kept out of TraceArgs, whose layout the
// whole-ID kernel's code generation is sensitive to (profiles/r01_ray_split_ab.log).
constexpr int kPeerTotalsOffset = 16;   // ints
__device__ __forceinline__ const PeerTotals *peer_totals_of(const TraceArgs &A)
{
    return reinterpret_cast<const PeerTotals *>(A.work_counter + kPeerTotalsOffset);
}
// SM-affine chunk order (NBT_SM_AFFINE = number of homes, experiment): perspective j belongs
// to home j mod H; a warp first takes chunks of the home of its SM (smid mod H) -- so the
// warps of one SM walk neighbouring tiles of the same frustum at the same time and share
// its map lines in L1 -- and then steals from the other homes in order.
#ifndef NBT_SM_AFFINE
#define NBT_SM_AFFINE 0
#endif
constexpr int kHomes = NBT_SM_AFFINE;
constexpr int kHomeCounterOffset = 128;  // ints: one counter per home
__device__ __forceinline__ int next_chunk_affine(const TraceArgs &A)
{
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int cpp = A.chunks_per_persp;
    const int n = A.total_chunks / cpp;
    const int homes = n < kHomes ? n : kHomes;
    const int h0 = (int)(smid % (unsigned)homes);
    for (int t = 0; t < homes; ++t) {
        const int h = h0 + t < homes ? h0 + t : h0 + t - homes;
        int *ctr = A.work_counter + kHomeCounterOffset + h;
        const int per = ((n - h + homes - 1) / homes) * cpp;   // chunks of home h
        if (*(volatile int *)ctr >= per) continue;
        const int k = atomicAdd(ctr, 1);
        if (k < per) return (h + homes * (k / cpp)) * cpp + k % cpp;
    }
    return A.total_chunks;
}

// Chunk index -> (perspective, first slot) in the NBT_CHUNK_ORDER order.
__device__ __forceinline__ void decode_chunk(const TraceArgs &A, int ch, int &q_j, int &q_next)
{
    if (NBT_CHUNK_ORDER == 1) {
        // position-major: top and bottom rows of tiles first, the middle rows last
        const int n = A.total_chunks / A.chunks_per_persp;
        const int pp = ch / n;
        q_j = ch - pp * n;
        const int qq = (pp & 1) ? A.chunks_per_persp - 1 - (pp >> 1) : (pp >> 1);
        q_next = qq * A.chunk;
    } else {
        q_j = ch / A.chunks_per_persp;
        q_next = (ch - q_j * A.chunks_per_persp) * A.chunk;
    }
}

// Grab g of the work counter -> the slot range [q_next, q_end) of perspective q_j; false once the
// work is out.  The launch's last chunks (from split_from on, NBT_SPLIT_TAIL per resident warp) are
// handed out as two halves, so the end of the launch waits on half chunks.
__device__ __forceinline__ bool take_grab(const TraceArgs &A, int g, int &q_j, int &q_next, int &q_end)
{
    if (g >= A.total_grabs) return false;
    int ch = g, len = A.chunk, half = 0;
    if (g >= A.split_from) {
        const int h = g - A.split_from;
        ch = A.split_from + (h >> 1);
        len = A.chunk >> 1;
        half = h & 1;
    }
    decode_chunk(A, ch, q_j, q_next);
    q_next += half * len;
    q_end = min(q_next + len, A.slots);
    return true;
}

// REC instance (nbt_debug_id_rays): the per-ray record array lives in the same buffer.
constexpr int kRecordOffset = 64;       // ints (after the peer totals)
static_assert(kPeerTotalsOffset * 4 + sizeof(PeerTotals) <= kRecordOffset * 4, "record after the peer totals");
__device__ __forceinline__ uint32_t *record_of(const TraceArgs &A)
{
    return *reinterpret_cast<uint32_t *const *>(A.work_counter + kRecordOffset);
}

// Map slot -> lattice offsets (mi, mk) = (2i-(W-1), 2kk-(H-1)) or a corner ray.
__device__ __forceinline__ bool slot_ray(const TraceArgs &T, int slot, int &mi, int &mk, int &corner)
{
    corner = -1;
    int i, kk;
    if (slot >= T.n_tile_slots) {
        corner = slot - T.n_tile_slots;
        return true;
    }
    if (T.tiled) {
        int tile = slot >> 5, l = slot & 31;
        int ty = tile / T.Wt, tx = tile - ty * T.Wt;
        i = tx * kTileW + (l & (kTileW - 1));
        kk = ty * kTileH + l / kTileW;
        if (i >= T.W || kk >= T.H) return false;
    } else {
        kk = slot / T.W;
        i = slot - kk * T.W;
    }
    mi = 2 * i - (T.W - 1);
    mk = 2 * kk - (T.H - 1);
    return true;
}

// Ray index k (Q27 order: row-major lattice, then the corner rays) of a (non-shard) slot.
__device__ __forceinline__ int ray_index_of_slot(const TraceArgs &T, int slot)
{
    int mi = 0, mk = 0, corner = -1;
    slot_ray(T, slot, mi, mk, corner);
    if (corner >= 0) return T.W * T.H + corner;
    return ((mk + T.H - 1) >> 1) * T.W + ((mi + T.W - 1) >> 1);
}

// REC: ray k of perspective j closed with these counts (n_U, n_F, n_O, lookups, stop).
__device__ __forceinline__ void record_ray(const TraceArgs &T, int j, int slot, uint32_t u, uint32_t f, uint32_t o,
                                           uint32_t l)
{
    const int ne = T.W * T.H + (T.add_corners ? 4 : 0);
    uint32_t *r = record_of(T) + 5 * ((size_t)j * ne + ray_index_of_slot(T, slot));
    r[0] = u; r[1] = f; r[2] = o; r[3] = l; r[4] = o;    // n_O in {0, 1} is the stop flag
}

// Walk segment of a ray: both ends on the Q16 lattice (modular arithmetic: the true
// values lie inside (-2^30, 2^30), checked per perspective; Q19).
__device__ __forceinline__ void ray_segment(const int f[18], int mi, int mk, int corner, int o[3], int e[3])
{
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        uint32_t v;
        if (corner < 0) {
            v = (uint32_t)f[k] + (uint32_t)f[3 + k] + (uint32_t)mi * (uint32_t)f[6 + k] +
                (uint32_t)mk * (uint32_t)f[9 + k];
        } else {
            uint32_t rc = (uint32_t)f[12 + k], uc = (uint32_t)f[15 + k];
            v = (uint32_t)f[k] + (uint32_t)f[3 + k] + ((corner & 1) ? rc : 0u - rc) + ((corner & 2) ? uc : 0u - uc);
        }
        o[k] = f[k];
        e[k] = (int)v;
    }
}


// Warp-cooperative flush (all 32 lanes call it): every lane with `fl` set adds its counts
// to perspective jl's totals and zeroes them; lanes with the same jl are summed first, so
// each (perspective, counter) takes one atomic per warp.  u, f, o, l are summed in 32 bits
// (bounded by the perspective's total), the Eq. 2 gain (63x larger) in 64.
template <bool GAIN>
__device__ __forceinline__ void flush_counts_warp(unsigned long long *totals, int jl, Counts &c, bool fl, int lane)
{
    const unsigned full = 0xffffffffu;
    unsigned fm = __ballot_sync(full, fl && jl >= 0);
    while (fm) {
        const int leader = __ffs(fm) - 1;
        const int pj = __shfl_sync(full, jl, leader);
        const bool mine = fl && jl == pj;
        const unsigned grp = __ballot_sync(full, mine);
        const uint32_t su = __reduce_add_sync(full, mine ? c.u : 0u);
        const uint32_t sf = __reduce_add_sync(full, mine ? c.f : 0u);
        const uint32_t so = __reduce_add_sync(full, mine ? c.o : 0u);
        const uint32_t sl = __reduce_add_sync(full, mine ? c.l : 0u);
        unsigned long long sg = 0;
        if (GAIN) {
            sg = mine ? (unsigned long long)c.g : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(full, sg, o);
        }
        if (lane == leader) {
            unsigned long long *t = totals + kTotals * (size_t)pj;
            if (su) atomicAdd(t + 0, (unsigned long long)su);
            if (sf) atomicAdd(t + 1, (unsigned long long)sf);
            if (so) atomicAdd(t + 2, (unsigned long long)so);
            if (sl) atomicAdd(t + 3, (unsigned long long)sl);
            if (GAIN && sg) atomicAdd(t + 4, sg);
        }
        if (mine) c = Counts{0, 0, 0, 0, 0};
        fm &= ~grp;
    }
}

// The same flush into every rank's totals (the ray split's all-reduce fused into the walk).
template <bool GAIN>
__device__ __forceinline__ void flush_counts_warp_peer(const PeerTotals *pt, int jl, Counts &c, bool fl, int lane)
{
    const unsigned full = 0xffffffffu;
    unsigned fm = __ballot_sync(full, fl && jl >= 0);
    while (fm) {
        const int leader = __ffs(fm) - 1;
        const int pj = __shfl_sync(full, jl, leader);
        const bool mine = fl && jl == pj;
        const unsigned grp = __ballot_sync(full, mine);
        const uint32_t su = __reduce_add_sync(full, mine ? c.u : 0u);
        const uint32_t sf = __reduce_add_sync(full, mine ? c.f : 0u);
        const uint32_t so = __reduce_add_sync(full, mine ? c.o : 0u);
        const uint32_t sl = __reduce_add_sync(full, mine ? c.l : 0u);
        unsigned long long sg = 0;
        if (GAIN) {
            sg = mine ? (unsigned long long)c.g : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(full, sg, o);
        }
        if (lane == leader) {
            for (int d = 0; d < pt->n; ++d) {       // every rank's totals, through the peer mappings
                unsigned long long *t = pt->t[d] + kTotals * (size_t)pj;
                if (su) atomicAdd(t + 0, (unsigned long long)su);
                if (sf) atomicAdd(t + 1, (unsigned long long)sf);
                if (so) atomicAdd(t + 2, (unsigned long long)so);
                if (sl) atomicAdd(t + 3, (unsigned long long)sl);
                if (GAIN && sg) atomicAdd(t + 4, sg);
            }
        }
        if (mine) c = Counts{0, 0, 0, 0, 0};
        fm &= ~grp;
    }
}

// Prepare the ray in `slot` of perspective j (frame, segment, DDA set-up, grid
// entry).  Returns false if the slot is a tile hole or the ray ends without entering
// the grid (its Unknown visits are then added to the totals directly).
// Unknown visits of a ray that never enters the grid, in a ray shard: into every rank's totals
// for the fused ray split (like the walked rays' flushes), else into the call's totals.  Rare,
// so kept out of line (the shard kernel's register budget).
__device__ __noinline__ void add_unknown_shard(const TraceArgs &A, int j, uint32_t pre)
{
    const PeerTotals *pt = peer_totals_of(A);
    const int nd = pt->n > 0 ? pt->n : 1;
    for (int d = 0; d < nd; ++d) {
        unsigned long long *t = (pt->n > 0 ? pt->t[d] : A.totals) + kTotals * (size_t)j;
        atomicAdd(t, (unsigned long long)pre);
        atomicAdd(t + 4, 63ull * pre);
    }
}

template <typename T, int L, int VB, bool SHARD, bool REC = false>
__device__ __forceinline__ bool prep_ray(const TraceArgs &A, int j, int slot, Walk<T> &w)
{
    int mi = 0, mk = 0, corner = -1;
    if (!slot_ray(A, slot, mi, mk, corner)) return false;
    const int4 *fp = reinterpret_cast<const int4 *>(A.frames + (size_t)j * kFrameInts);
    int4 q0 = __ldg(fp), q1 = __ldg(fp + 1), q2 = __ldg(fp + 2), q3 = __ldg(fp + 3), q4 = __ldg(fp + 4);
    const int f[18] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x,
                       q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w, q4.x, q4.y};
    int o[3], e[3];
    ray_segment(f, mi, mk, corner, o, e);
    walk_setup(w, o, e);
    if (walk_enter<T, L, false, idx_shift<L, VB>()>(w, A.m, nullptr, nullptr, 0)) {
        if (A.m.policy == NBT_OUTSIDE_UNKNOWN) {
            if (SHARD) {
                add_unknown_shard(A, j, w.pre);
            } else {
                atomicAdd(A.totals + kTotals * (size_t)j, (unsigned long long)w.pre);
                atomicAdd(A.totals + kTotals * (size_t)j + 4, 63ull * w.pre);
            }
        }
        if (REC) record_ray(A, j, slot, A.m.policy == NBT_OUTSIDE_UNKNOWN ? w.pre : 0u, 0u, 0u, 0u);
        return false;
    }
    return true;
}

// Per-warp queue of prepared walks in shared memory (structure of arrays, one column
// per entry, so 32 lanes touching 32 entries hit 32 banks).
// A queue holds the rays of ONE fill (one 32-slot unit of one perspective: the warp-uniform
// q_j), and every queued ray entered the grid, so its outside visits equal its entry step
// (pre == s0): neither is stored.  32-bit decision terms travel in int2 columns (one 8-byte
// shared access per pair of fields and lane: 6 + 6 instead of 14 + 14 per ray).
template <typename T>
struct WalkQueue {
    T q[3][32];
    T a[3][32];
    uint32_t idx[32];
    int d[3][32];                // linear: dX, dY, ndZ; Morton: rx, ry, rz
    uint32_t xinv[32];           // Morton only
    int n[32], s0[32];
};
template <>
struct WalkQueue<int> {
    int2 qq[32];                 // (qxy, qxz)
    int2 qa[32];                 // (qyz, ax)
    int2 aa[32];                 // (ay, az)
    int2 id[32];                 // (idx, d0)
    int2 dd[32];                 // (d1, d2); linear: dX, dY, ndZ; Morton: rx, ry, rz
    int2 ns[32];                 // (n, s0)
    uint32_t xinv[32];           // Morton only
};
// REC instance: the queue also carries each prepared ray's slot.
template <typename T>
struct WalkQueueRec : WalkQueue<T> {
    int slot[32];
};

template <typename T, int L, typename Queue>
__device__ __forceinline__ void queue_put(Queue &Q, int i, const Walk<T> &w)
{
    const int d0 = L == kLayoutMorton ? (int)w.rx : w.dX, d1 = L == kLayoutMorton ? (int)w.ry : w.dY,
              d2 = L == kLayoutMorton ? (int)w.rz : w.ndZ;
    if constexpr (sizeof(T) == 4) {
        Q.qq[i] = make_int2(w.qxy, w.qxz);
        Q.qa[i] = make_int2(w.qyz, w.ax);
        Q.aa[i] = make_int2(w.ay, w.az);
        Q.id[i] = make_int2((int)w.idx, d0);
        Q.dd[i] = make_int2(d1, d2);
        Q.ns[i] = make_int2(w.n, w.s0);
    } else {
        Q.q[0][i] = w.qxy; Q.q[1][i] = w.qxz; Q.q[2][i] = w.qyz;
        Q.a[0][i] = w.ax; Q.a[1][i] = w.ay; Q.a[2][i] = w.az;
        Q.idx[i] = w.idx;
        Q.d[0][i] = d0; Q.d[1][i] = d1; Q.d[2][i] = d2;
        Q.n[i] = w.n; Q.s0[i] = w.s0;
    }
    if (L == kLayoutMorton) Q.xinv[i] = w.xinv;
}

template <typename T, int L, typename Queue>
__device__ __forceinline__ void queue_get(const Queue &Q, int i, Walk<T> &w)
{
    int d0, d1, d2;
    if constexpr (sizeof(T) == 4) {
        const int2 qq = Q.qq[i], qa = Q.qa[i], aa = Q.aa[i], id = Q.id[i], dd = Q.dd[i], ns = Q.ns[i];
        w.qxy = qq.x; w.qxz = qq.y; w.qyz = qa.x;
        w.ax = qa.y; w.ay = aa.x; w.az = aa.y;
        w.idx = (uint32_t)id.x;
        d0 = id.y; d1 = dd.x; d2 = dd.y;
        w.n = ns.x; w.s0 = ns.y;
    } else {
        w.qxy = Q.q[0][i]; w.qxz = Q.q[1][i]; w.qyz = Q.q[2][i];
        w.ax = Q.a[0][i]; w.ay = Q.a[1][i]; w.az = Q.a[2][i];
        w.idx = Q.idx[i];
        d0 = Q.d[0][i]; d1 = Q.d[1][i]; d2 = Q.d[2][i];
        w.n = Q.n[i]; w.s0 = Q.s0[i];
    }
    if (L == kLayoutMorton) {
        w.rx = (uint32_t)d0; w.ry = (uint32_t)d1; w.rz = (uint32_t)d2;
        w.xinv = Q.xinv[i];
    } else {
        w.dX = d0; w.dY = d1; w.ndZ = d2;
    }
    w.s = w.s0; w.pre = (uint32_t)w.s0; w.nf = 0; w.ng = 0;   // queued rays entered the grid: pre == s0
    w.nax = -w.ax;
}

// Resident blocks per SM the register allocation must allow: 4 (64 registers, 32 warps) for
// the 32-bit 2-bit-store instance that every config uses -- measured 5-10% faster than the
// unconstrained 92 registers (2 blocks) -- 3 for the 8-bit store and 2 for the 64-bit-term
// instances (long rays), which would spill at fewer registers.
#ifndef NBT_TRACE_MIN_BLOCKS
#define NBT_TRACE_MIN_BLOCKS 0
#endif
template <typename T, int VB>
constexpr int trace_min_blocks()
{
    // resident warps per SM the register budget must allow: 32 (64 registers), 24 or 16
    return NBT_TRACE_MIN_BLOCKS > 0 ? NBT_TRACE_MIN_BLOCKS
                                    : (sizeof(T) == 8 ? 16 : (VB == kStoreProb ? 24 : 32)) / kWarpsPerBlock;
}

// REC = per-ray record instance (nbt_debug_id_rays): the same code, which also writes every
// closed ray's counts to the record array; a separate instance, so the production kernel's
// code is unchanged.
// LOCK: the lockstep walk (NBT_OPT_TRACE_REFILL_MIN = 32, the default) specialised -- a tile's rays
// prepared straight into the lanes' walks (no queue, no shared memory) and the batch loop left when
// no lane walks (one vote).  LOCK = false: the general form with per-lane refills from a queue.
template <typename T, int L, int VB, int K, bool PIPE, bool SHARD, bool REC = false, bool LOCK = false>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, trace_min_blocks<T, VB>()) k_id_trace(TraceArgs A)
{
    constexpr bool CYCLE = PIPE && VB != kStoreProb;     // in-place pipeline (batch_cycle)
    static_assert((CYCLE ? 2 * K : K) <= kBorder, "look-ahead must stay inside the sentinel shell");
    static_assert(!(REC && (SHARD || CYCLE)), "the record instance is the whole-ID, unpipelined walk");
    using Queue = std::conditional_t<LOCK, char, std::conditional_t<REC, WalkQueueRec<T>, WalkQueue<T>>>;
    __shared__ Queue queues[LOCK ? 1 : kWarpsPerBlock];
    Queue &Q = queues[LOCK ? 0 : (threadIdx.x >> 5)];
    constexpr bool TAB = kDdaTable && sizeof(T) == 4 && L == kLayoutLinear && !CYCLE;
    __shared__ int4 step_tab[TAB ? kWarpsPerBlock * 96 : 1];
    // this lane's z-step entry: step_tab[warp][2][lane] (x, y entries 64 and 32 int4 below)
    const uint32_t tz = (uint32_t)__cvta_generic_to_shared(step_tab) +
                        (TAB ? (uint32_t)(((threadIdx.x >> 5) * 96 + 64 + (threadIdx.x & 31)) * 16) : 0u);
    int my_slot = 0;                         // REC: slot of this lane's ray
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lanes_below = (1u << lane) - 1u;
    int q_j = 0, q_next = 0, q_end = 0;      // warp-uniform chunk cursor
    bool q_done = false;
    int qhead = 0, qcount = 0;               // warp-uniform prepared-walk queue
    int q_jq = 0;                            // ... and the perspective of its rays
    Walk<T> w;
    Batch<K> b0;
    int have = 0;                            // this lane walks a ray (an int: no predicate byte packing)
    int jl = -1;                             // perspective of this lane's accumulators
    Counts c{0, 0, 0, 0, 0};
    // idle lanes that end the batch loop (32 once the work is out).  Default 32: a warp takes the
    // next 32 prepared rays (one 8x4 pixel tile) only when all its lanes are idle, so a tile's rays
    // start together and walk at the same depth -- a warp request touches fewer map lines, and a
    // tile's rays have similar lengths (88% of the lane-visit slots busy on D, oracle walks).
    // Measured against per-lane refills at 4-24 idle lanes (profiles/r02_s3_refill*.log): B -4%,
    // C' -4.6%, D +-0.
    int thr = A.min_refill;
    for (;;) {
        // the walk: batches until enough lanes are idle (min_refill = 1: as soon as any is)
        unsigned need;
        for (;;) {
            if (have) {
                if (CYCLE) {
                    // b0 holds visits s..s+K-1 (issued at the ray's start or by the last cycle)
                    uint32_t bits;
                    if (w.n - w.s + 1 > K) {
                        bits = batch_cycle<T, L, VB, K>(w, A.m, b0);
                    } else {
                        bits = batch_bits<VB, K>(b0);
                    }
                    if (batch_finish<T, VB, K>(w, bits, 0u, b0, A.m.policy, c)) have = 0;
                } else {
                    batch_issue<T, L, VB, K, TAB>(w, A.m, b0, tz);
                    const Counts before = c;
                    if (batch_consume<T, VB, K>(w, b0, A.m.policy, c)) {
                        have = 0;
                        if (REC)
                            record_ray(A, jl, my_slot, c.u - before.u, c.f - before.f, c.o - before.o,
                                       c.l - before.l);
                    }
                }
            }
            if constexpr (LOCK) {
                if (!__any_sync(full, have)) break;
            } else {
                need = __ballot_sync(full, !have);
                if (__popc(need) >= thr) break;
            }
        }
        if constexpr (LOCK) {
            // every lane is idle: the next 32-ray unit, prepared straight into the lanes' walks
            for (;;) {
                if (q_next >= q_end) {
                    int ch = 0;
                    if (lane == 0) ch = kHomes > 0 ? next_chunk_affine(A) : atomicAdd(A.work_counter, 1);
                    ch = __shfl_sync(full, ch, 0);
                    if (!take_grab(A, ch, q_j, q_next, q_end)) { q_done = true; break; }
                    if (__ldg(A.frames + (size_t)q_j * kFrameInts + 18) != 0) q_next = q_end;   // invalid
                    continue;
                }
                const int avail = min(32, q_end - q_next);
                int slot0 = q_next, valid = avail;
                if (SHARD) {
                    if (q_next < A.local_tile_slots) {
                        slot0 = ((q_next >> 5) * A.ray_world + A.ray_rank) << 5;
                        valid = min(avail, A.n_tile_slots - slot0);
                    } else {
                        slot0 = q_next - A.local_tile_slots + A.n_tile_slots;
                    }
                }
                const bool ok = lane < valid && prep_ray<T, L, VB, SHARD, REC>(A, q_j, slot0 + lane, w);
                q_next += avail;
                if (!__any_sync(full, ok)) continue;
                // lanes moving to another perspective flush their counts (warp-combined)
                const bool fl = ok && q_j != jl;
                if (SHARD && peer_totals_of(A)->n > 0)
                    flush_counts_warp_peer<VB == kStoreProb>(peer_totals_of(A), jl, c, fl, lane);
                else
                    flush_counts_warp<VB == kStoreProb>(A.totals, jl, c, fl, lane);
                if (ok) {
                    jl = q_j;
                    have = 1;
                    if constexpr (REC) my_slot = slot0 + lane;
                    if (TAB) table_put(tz, w);
                    if (CYCLE) batch_issue<T, L, VB, K>(w, A.m, b0);
                }
                break;
            }
            if (q_done) break;                   // every lane idle and no work left
            continue;
        } else {
            // all 32 lanes prepare up to 32 rays at once, so the set-up runs converged
            while (qcount == 0 && !q_done) {
                if (q_next >= q_end) {
                    int ch = 0;
                    if (lane == 0) ch = kHomes > 0 ? next_chunk_affine(A) : atomicAdd(A.work_counter, 1);
                    ch = __shfl_sync(full, ch, 0);
                    if (!take_grab(A, ch, q_j, q_next, q_end)) { q_done = true; break; }
                    if (__ldg(A.frames + (size_t)q_j * kFrameInts + 18) != 0) q_next = q_end;   // invalid
                    continue;
                }
                const int avail = min(32, q_end - q_next);
                int slot0 = q_next, valid = avail;
                if (SHARD) {
                    // ray shard: local 32-slot unit u -> lattice unit u * ray_world + ray_rank
                    // (chunks are whole units), then shard 0's corner rays (a separate
                    // instance, so the whole-ID kernel's code is unchanged)
                    if (q_next < A.local_tile_slots) {
                        slot0 = ((q_next >> 5) * A.ray_world + A.ray_rank) << 5;
                        valid = min(avail, A.n_tile_slots - slot0);
                    } else {
                        slot0 = q_next - A.local_tile_slots + A.n_tile_slots;
                    }
                }
                Walk<T> t;
                const bool ok = lane < valid && prep_ray<T, L, VB, SHARD, REC>(A, q_j, slot0 + lane, t);
                q_next += avail;
                const unsigned vm = __ballot_sync(full, ok);
                if (ok) queue_put<T, L>(Q, __popc(vm & lanes_below), t);
                q_jq = q_j;                                        // the queue's perspective
                if constexpr (REC) {
                    if (ok) Q.slot[__popc(vm & lanes_below)] = slot0 + lane;
                }
                __syncwarp();
                qhead = 0;
                qcount = __popc(vm);
            }
            if (qcount) {
                const int rank = __popc(need & lanes_below);
                const int take = min(__popc(need), qcount);
                int j = -1;
                if (!have && rank < take) {
                    queue_get<T, L>(Q, qhead + rank, w);
                    j = q_jq;
                    if constexpr (REC) my_slot = Q.slot[qhead + rank];
                }
                // lanes moving to another perspective flush their counts, one atomic per
                // counter per (warp, perspective): many lanes of a warp hold the same one
                const bool fl = j >= 0 && j != jl;
                if (SHARD && peer_totals_of(A)->n > 0)
                    flush_counts_warp_peer<VB == kStoreProb>(peer_totals_of(A), jl, c, fl, lane);
                else
                    flush_counts_warp<VB == kStoreProb>(A.totals, jl, c, fl, lane);
                if (j >= 0) {
                    jl = j;
                    have = 1;
                    if (TAB) table_put(tz, w);
                    if (CYCLE) batch_issue<T, L, VB, K>(w, A.m, b0);
                }
                qhead += take;
                qcount -= take;
                __syncwarp();
            }
        }
        if (q_done && qcount == 0) {
            if (!__any_sync(full, have)) break;  // every lane idle and no work left
            thr = 32;                            // let the last walks finish
        }
    }
    // residual counts, once per lane (the warp-combined form measured ~2% slower here)
    if (jl >= 0 && SHARD && peer_totals_of(A)->n > 0) {
        const PeerTotals *pt = peer_totals_of(A);
        for (int d = 0; d < pt->n; ++d) {
            unsigned long long *t = pt->t[d] + kTotals * (size_t)jl;
            if (c.u) atomicAdd(t + 0, (unsigned long long)c.u);
            if (c.f) atomicAdd(t + 1, (unsigned long long)c.f);
            if (c.o) atomicAdd(t + 2, (unsigned long long)c.o);
            if (c.l) atomicAdd(t + 3, (unsigned long long)c.l);
            if (VB == kStoreProb && c.g) atomicAdd(t + 4, (unsigned long long)c.g);
        }
    } else if (jl >= 0) {
        unsigned long long *t = A.totals + kTotals * (size_t)jl;
        if (c.u) atomicAdd(t + 0, (unsigned long long)c.u);
        if (c.f) atomicAdd(t + 1, (unsigned long long)c.f);
        if (c.o) atomicAdd(t + 2, (unsigned long long)c.o);
        if (c.l) atomicAdd(t + 3, (unsigned long long)c.l);
        if (VB == kStoreProb && c.g) atomicAdd(t + 4, (unsigned long long)c.g);
    }
}

// ------------------------------------------------------------ finalize (a8)

__global__ void k_id_finalize(FrameArgs A, const int32_t *__restrict__ frames,
                              const unsigned long long *__restrict__ totals, double g_u, double g_f, double g_o,
                              int prob, double n_e, double *__restrict__ xyz_out, double *__restrict__ gain_out,
                              unsigned long long *__restrict__ counts_out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const double *pp = A.persp + 3 * (size_t)(A.first + (size_t)i * A.stride);
    xyz_out[3 * (size_t)i + 0] = pp[0];
    xyz_out[3 * (size_t)i + 1] = pp[1];
    xyz_out[3 * (size_t)i + 2] = pp[2];
    const unsigned long long *t = totals + kTotals * (size_t)i;
    unsigned long long tu = t[0], tf = t[1], to = t[2], tl = t[3], tg = t[4];
    // per-state gains (Q26) or, with per-voxel probabilities, the exact Eq. 2 sum (Q32)
    double g = prob ? __ddiv_rn((double)tg, __dmul_rn(63.0, n_e))
                    : __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)tu, g_u), __dmul_rn((double)tf, g_f)),
                                          __dmul_rn((double)to, g_o)),
                                n_e);
    if (frames[(size_t)i * kFrameInts + 18] != 0) g = __longlong_as_double(0x7ff8000000000000LL);   // NaN
    gain_out[i] = g;
    if (counts_out) {
        counts_out[4 * (size_t)i + 0] = tu;
        counts_out[4 * (size_t)i + 1] = tf;
        counts_out[4 * (size_t)i + 2] = to;
        counts_out[4 * (size_t)i + 3] = tl;
    }
}

// The finalize of a shard fused with the all-gather: row i of this call (perspective
// first + i*stride of the call's array) is row row0 + first + i*stride of the whole cloud, written (same values as k_id_finalize) into every
// destination's row buffer -- the other ranks' buffers are peer mappings, so the stores
// travel over NVLink/NVSwitch.
__global__ void k_id_finalize_gather(FrameArgs A, const int32_t *__restrict__ frames,
                                     const unsigned long long *__restrict__ totals, double g_u, double g_f,
                                     double g_o, int prob, double n_e, int32_t row0,
                                     const __grid_constant__ GatherDst dst)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const size_t src = (size_t)A.first + (size_t)i * A.stride;
    const size_t row = (size_t)row0 + src;
    const double *pp = A.persp + 3 * src;
    const double px = pp[0], py = pp[1], pz = pp[2];
    const unsigned long long *t = totals + kTotals * (size_t)i;
    const unsigned long long tu = t[0], tf = t[1], to = t[2], tl = t[3], tg = t[4];
    double g = prob ? __ddiv_rn((double)tg, __dmul_rn(63.0, n_e))
                    : __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn((double)tu, g_u), __dmul_rn((double)tf, g_f)),
                                          __dmul_rn((double)to, g_o)),
                                n_e);
    if (frames[(size_t)i * kFrameInts + 18] != 0) g = __longlong_as_double(0x7ff8000000000000LL);   // NaN
    for (int d = 0; d < dst.n; ++d) {
        double *x = dst.xyz[d] + 3 * row;
        x[0] = px; x[1] = py; x[2] = pz;
        dst.gain[d][row] = g;
        unsigned long long *c = dst.counts[d] + 4 * row;
        c[0] = tu; c[1] = tf; c[2] = to; c[3] = tl;
    }
}

// ------------------------------------------------------------ debug hooks

// Per-ray walk of an explicit Q16 segment, recording every visited voxel; the same
// Walk / walk_step / walk_enter code as k_id_trace, one voxel at a time.
template <typename T, int L, int VB>
__global__ void k_debug_trace(MapView m, const int32_t *__restrict__ o, const int32_t *__restrict__ e, int n_rays,
                              int max_visits, int32_t *ijk, uint8_t *code, int32_t *len, uint32_t *counts)
{
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    int oo[3] = {o[3 * r], o[3 * r + 1], o[3 * r + 2]};
    int ee[3] = {e[3 * r], e[3 * r + 1], e[3 * r + 2]};
    Walk<T> w;
    walk_setup(w, oo, ee);
    int32_t *ri = ijk + (size_t)r * max_visits * 3;
    uint8_t *rc = code + (size_t)r * max_visits;
    Counts c{0, 0, 0, 0, 0};
    int visits;
    if (walk_enter<T, L, true, idx_shift<L, VB>()>(w, m, ri, rc, max_visits)) {
        if (m.policy == NBT_OUTSIDE_UNKNOWN) c.u += w.pre;
        visits = w.n + 1;
    } else {
        for (;;) {
            const uint32_t ib = L == kLayoutLinear ? w.idx : (w.idx << 1);   // 2-bit store: bit offset
            const uint32_t cd = VB == kStore2 ? code_of(__ldg(m.words + (ib >> 5)), ib)
                                              : __ldg(reinterpret_cast<const uint8_t *>(m.words) + w.idx) & 3u;
            if (w.s < max_visits) {
                ri[3 * w.s] = w.vx; ri[3 * w.s + 1] = w.vy; ri[3 * w.s + 2] = w.vz;
                rc[w.s] = cd == 3u ? 255 : (uint8_t)cd;
            }
            if (cd >= 2u) {
                walk_close_stop(w, m.policy, cd, w.s, w.nf, 0u, c);
                if (cd == 2u) {
                    visits = w.s + 1;
                } else {   // record the outside tail too
                    for (int s = w.s + 1; s <= w.n; ++s) {
                        walk_step<T, L, true>(w, m);
                        if (s < max_visits) {
                            ri[3 * s] = w.vx; ri[3 * s + 1] = w.vy; ri[3 * s + 2] = w.vz;
                            rc[s] = 255;
                        }
                    }
                    visits = w.n + 1;
                }
                break;
            }
            w.nf += cd;
            if (w.s == w.n) {
                walk_close_end(w, m.policy, w.nf, 0u, c);
                visits = w.n + 1;
                break;
            }
            walk_step<T, L, true>(w, m);
            w.s++;
        }
    }
    len[r] = visits;
    counts[4 * r + 0] = c.u; counts[4 * r + 1] = c.f; counts[4 * r + 2] = c.o; counts[4 * r + 3] = c.l;
}

__global__ void k_debug_frames(FrameArgs A, int32_t *out)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const double *pp = A.persp + 3 * (size_t)i;
    double p[3] = {pp[0], pp[1], pp[2]};
    int f[18] = {0};
    int st = make_frame(A, p, f);
    for (int k = 0; k < 18; ++k) out[19 * (size_t)i + k] = st ? 0 : f[k];
    out[19 * (size_t)i + 18] = st;
}

MapView view_of(nbt_map m)
{
    MapView v;
    v.words = m->d_words;
    v.nx = m->desc.nx; v.ny = m->desc.ny; v.nz = m->desc.nz;
    v.px = (int)m->px;
    v.pxy = (int)(m->px * m->py);
    const uint32_t all = m->layout == kLayoutMorton ? ((1u << (3 * m->pbits)) - 1u) : 0u;
    v.mx = 0x09249249u & all;
    v.my = 0x12492492u & all;
    v.mz = 0x24924924u & all;
    v.policy = m->desc.outside_policy;
    return v;
}

FrameArgs frame_args(nbt_map m, const double *d_persp, int32_t first, int32_t stride, int32_t n, const double poi[3],
                     const nbt_camera &cam, double range)
{
    FrameArgs A;
    A.persp = d_persp; A.first = first; A.stride = stride; A.n = n;
    for (int k = 0; k < 3; ++k) { A.poi[k] = poi[k]; A.origin[k] = m->desc.origin[k]; }
    A.voxel_size = m->desc.voxel_size;
    A.range = range;
    A.cam = cam;
    return A;
}

// Conservative bound (voxels) on |D_a| of every ray of a camera: the longest ray of the
// frustum (its far-plane corner) plus rounding.
double max_ray_voxels(const nbt_camera &cam, double range, double voxel_size)
{
    double rs = range / voxel_size;
    double ex = (cam.width - 1) / (2.0 * cam.fx), ey = (cam.height - 1) / (2.0 * cam.fy);
    if (cam.add_corners) {
        ex = fmax(ex, cam.tan_half_fov_h);
        ey = fmax(ey, cam.tan_half_fov_v);
    }
    return rs * sqrt(1.0 + ex * ex + ey * ey) * 1.001 + 2.0;
}

// The kernel instances: [ray shard][wide][layout][store: 2-bit, byte, byte + gain].
// [lock][shard][wide][layout][store]
#define NBT_TRACE_ROW(T, L, S, LK)                                                                                 \
    {k_id_trace<T, L, kStore2, kBatchK, kPipe, S, false, LK>, k_id_trace<T, L, kStoreByte, kBatchK, kPipe, S, false, LK>, \
     k_id_trace<T, L, kStoreProb, kBatchK, kPipe, S, false, LK>}
#define NBT_TRACE_SET(S, LK)                                                              \
    {{NBT_TRACE_ROW(int, kLayoutLinear, S, LK), NBT_TRACE_ROW(int, kLayoutMorton, S, LK)}, \
     {NBT_TRACE_ROW(long long, kLayoutLinear, S, LK), NBT_TRACE_ROW(long long, kLayoutMorton, S, LK)}}
using TraceFn = void (*)(TraceArgs);
const TraceFn kTraceFns[2][2][2][2][3] = {{NBT_TRACE_SET(false, false), NBT_TRACE_SET(true, false)},
                                          {NBT_TRACE_SET(false, true), NBT_TRACE_SET(true, true)}};
#undef NBT_TRACE_SET
#undef NBT_TRACE_ROW
// The per-ray record instances (nbt_debug_id_rays): [lock][wide][layout][store], unpipelined.
#define NBT_TRACE_REC_ROW(T, L, LK)                                                                 \
    {k_id_trace<T, L, kStore2, kBatchK, false, false, true, LK>,                                    \
     k_id_trace<T, L, kStoreByte, kBatchK, false, false, true, LK>,                                 \
     k_id_trace<T, L, kStoreProb, kBatchK, false, false, true, LK>}
#define NBT_TRACE_REC_SET(LK)                                                                \
    {{NBT_TRACE_REC_ROW(int, kLayoutLinear, LK), NBT_TRACE_REC_ROW(int, kLayoutMorton, LK)}, \
     {NBT_TRACE_REC_ROW(long long, kLayoutLinear, LK), NBT_TRACE_REC_ROW(long long, kLayoutMorton, LK)}}
const TraceFn kTraceRecFns[2][2][2][3] = {NBT_TRACE_REC_SET(false), NBT_TRACE_REC_SET(true)};
#undef NBT_TRACE_REC_SET
#undef NBT_TRACE_REC_ROW

using DebugFn = void (*)(MapView, const int32_t *, const int32_t *, int, int, int32_t *, uint8_t *, int32_t *,
                         uint32_t *);
#define NBT_DEBUG_ROW(T, L) \
    {k_debug_trace<T, L, kStore2>, k_debug_trace<T, L, kStoreByte>, k_debug_trace<T, L, kStoreProb>}
const DebugFn kDebugFns[2][2][3] = {{NBT_DEBUG_ROW(int, kLayoutLinear), NBT_DEBUG_ROW(int, kLayoutMorton)},
                                    {NBT_DEBUG_ROW(long long, kLayoutLinear), NBT_DEBUG_ROW(long long, kLayoutMorton)}};
#undef NBT_DEBUG_ROW

// Store kind of a map handle (index of the tables above).
int store_kind(nbt_map m) { return m->vbits == 2 ? 0 : (m->prob ? 2 : 1); }

}  // namespace

nbt_status launch_id(nbt_ctx ctx, nbt_map m, const IdLaunch &L)
{
    if (L.n == 0) return NBT_OK;
    nbt_status st;
    if ((st = ctx->frames.ensure((size_t)L.n * kFrameInts * 4))) return st;
    if ((st = ctx->totals.ensure((size_t)L.n * kTotals * 8))) return st;
    // totals the trace accumulates into (zeroed by k_persp_frames): the caller's array for a
    // ray shard, else scratch; the finalize reads the caller's summed totals when given
    unsigned long long *tot = L.d_totals_trace ? reinterpret_cast<unsigned long long *>(L.d_totals_trace)
                                               : ctx->totals.as<unsigned long long>();
    if ((st = ctx->counter.ensure((kHomeCounterOffset + (kHomes > 0 ? kHomes : 1)) * 4))) return st;
    static_assert(kRecordOffset * 4 + sizeof(void *) <= kHomeCounterOffset * 4, "home counters after the record");
    FrameArgs A = frame_args(m, L.d_persp, L.first, L.stride, L.n, L.poi, L.cam, L.range);
    int *counter = ctx->counter.as<int>();
    if (kHomes > 0)      // zeroed home counters (a memset node: valid inside a captured graph)
        NBT_CUDA(cudaMemsetAsync(counter + kHomeCounterOffset, 0, kHomes * 4, ctx->stream));
    {
        ProfScope ps(ctx, NBT_KERNEL_FRAMES);
        k_persp_frames<<<(L.n + 127) / 128, 128, 0, ctx->stream>>>(A, ctx->frames.as<int32_t>(),
                                                                    tot, counter,
                                                                    ctx->d_err);
        NBT_LAUNCHED(ctx);
    }

    TraceArgs T;
    T.m = view_of(m);
    T.frames = ctx->frames.as<int32_t>();
    T.totals = tot;
    T.work_counter = counter;
    T.W = L.cam.width; T.H = L.cam.height; T.add_corners = L.cam.add_corners ? 1 : 0;
    T.tiled = (T.W >= kTileW && T.H >= kTileH) ? 1 : 0;
    T.Wt = (T.W + kTileW - 1) / kTileW;
    int Ht = (T.H + kTileH - 1) / kTileH;
    T.n_tile_slots = T.tiled ? T.Wt * Ht * 32 : T.W * T.H;
    // ray shard (SURVEY 8(e) ray split): units of 32 lattice slots dealt round-robin
    const int units = (T.n_tile_slots + 31) / 32;
    T.ray_rank = L.ray_rank;
    T.ray_world = L.ray_world;
    T.local_tile_slots = L.ray_world == 1 ? T.n_tile_slots
                         : units > L.ray_rank ? ((units - L.ray_rank + L.ray_world - 1) / L.ray_world) * 32 : 0;
    T.slots = T.local_tile_slots + ((T.add_corners && L.ray_rank == 0) ? 4 : 0);
    const bool wide = max_ray_voxels(L.cam, L.range, m->desc.voxel_size) > kInt32MaxVoxels;
    const int sk = store_kind(m);
    const bool peer = L.peer_totals != nullptr && L.peer_totals->n > 0;
    if (L.ray_world > 1 || peer) {   // the SHARD instance reads its peer totals (n = 0: none)
        // device-to-device copy / memset only: both are valid graph nodes (no host source)
        if (peer)
            NBT_CUDA(cudaMemcpyAsync(counter + kPeerTotalsOffset, L.d_peer_totals, sizeof(PeerTotals),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
        else
            NBT_CUDA(cudaMemsetAsync(counter + kPeerTotalsOffset, 0, sizeof(PeerTotals), ctx->stream));
    }
    if (L.d_record)   // REC instance: where it writes the per-ray counts (debug entry, never captured)
        NBT_CUDA(cudaMemcpyAsync(counter + kRecordOffset, &L.d_record, sizeof(void *), cudaMemcpyHostToDevice,
                                 ctx->stream));
    const int lock = ctx->opt.refill_min >= 32;   // the lockstep instance (default) or per-lane refills
    const TraceFn fn = L.d_record ? kTraceRecFns[lock][wide][m->layout == kLayoutMorton][sk]
                                  : kTraceFns[lock][L.ray_world > 1 || peer][wide][m->layout == kLayoutMorton][sk];
    const int fi = lock * 12 + (wide ? 6 : 0) + (m->layout == kLayoutMorton ? 3 : 0) + sk;
    if (ctx->trace_blocks_per_sm == 0) {
        // smallest shared-memory carveout that holds the walk queues of the resident blocks,
        // so the rest of the SM's 256 KB stays L1 for the map lines
        // preferred shared-memory carveout (NBT_OPT_TRACE_CARVEOUT, default 25; -1 = driver)
        // (the lockstep instances hold no queue: the carveout applies to the refill instances)
        const int carve = ctx->opt.carveout;
        if (carve >= 0) {
            for (auto &lk : kTraceFns)
                for (auto &sh : lk)
                    for (auto &a : sh)
                        for (auto &b : a)
                            for (TraceFn f : b)
                                NBT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            for (auto &lk : kTraceRecFns)
                for (auto &a : lk)
                    for (auto &b : a)
                        for (TraceFn f : b)
                            NBT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
        }
        for (int k = 0; k < 24; ++k) {
            int b = 0;
            NBT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &b, kTraceFns[k / 12][0][(k / 6) & 1][(k / 3) & 1][k % 3], kWarpsPerBlock * 32, 0));
            ctx->trace_bps[k] = b > 0 ? b : 1;
        }
        ctx->trace_blocks_per_sm = ctx->trace_bps[12];
        if (ctx->opt.verbose) {
            fprintf(stderr, "libnbt: k_id_trace resident blocks/SM");
            for (int k = 0; k < 24; ++k) fprintf(stderr, " %d", ctx->trace_bps[k]);
            fprintf(stderr, " (carveout %d)\n", carve);
        }
    }
    const int bps = ctx->trace_bps[fi];
    long long resident_warps = (long long)ctx->num_sms * bps * kWarpsPerBlock;
    long long total_slots = (long long)L.n * T.slots;
    long long per = total_slots / (NBT_CHUNKS_PER_WARP * resident_warps);   // chunks per warp to aim for
    int chunk = (int)((per / 32) * 32);
    // smallest chunk per grab of the work counter (NBT_OPT_TRACE_CHUNK_MIN, default 64,
    // profiles/r01_chunk_flush.log)
    const int cmin = ctx->opt.chunk_min;
    chunk = chunk < cmin ? cmin : (chunk > NBT_CHUNK_MAX ? NBT_CHUNK_MAX : chunk);
    T.chunk = chunk;
    T.chunks_per_persp = (T.slots + chunk - 1) / chunk;
    long long tc = (long long)T.chunks_per_persp * L.n;
    if (tc >= (1ll << 31)) return fail(NBT_ERR_INVALID_ARG, "nbt_id_compute: too many rays in one call");
    T.total_chunks = (int)tc;
    // the last NBT_SPLIT_TAIL chunks per resident warp as half chunks (chunks of >= 64 slots)
    const long long tail = (long long)NBT_SPLIT_TAIL * resident_warps;
    T.split_from = (kHomes > 0 || chunk < 64 || tail == 0) ? T.total_chunks : (int)(tc > tail ? tc - tail : 0);
    T.total_grabs = T.split_from + 2 * (T.total_chunks - T.split_from);
    T.min_refill = ctx->opt.refill_min;   // NBT_OPT_TRACE_REFILL_MIN (profiles/r01_refill_sweep.log)
    long long want_blocks = (tc + kWarpsPerBlock - 1) / kWarpsPerBlock;
    long long max_blocks = (long long)ctx->num_sms * bps;
    int blocks = (int)(want_blocks < max_blocks ? want_blocks : max_blocks);
    if (blocks > 0 && !L.d_totals_final) {
        ProfScope ps(ctx, NBT_KERNEL_TRACE);
        fn<<<dim3(blocks), dim3(kWarpsPerBlock * 32), 0, ctx->stream>>>(T);
        NBT_LAUNCHED(ctx);
    }

    if (L.d_totals_trace || L.peer_totals) return NBT_OK;   // ray shard: partial totals only
    int ne = L.cam.width * L.cam.height + (L.cam.add_corners ? 4 : 0);
    ProfScope ps(ctx, NBT_KERNEL_FINALIZE);
    if (L.gather) {
        k_id_finalize_gather<<<(L.n + 127) / 128, 128, 0, ctx->stream>>>(
            A, ctx->frames.as<int32_t>(), tot, m->desc.gain[0], m->desc.gain[1], m->desc.gain[2], m->prob ? 1 : 0,
            (double)ne, L.gather_row0, *L.gather);
        NBT_LAUNCHED(ctx);
        return NBT_OK;
    }
    k_id_finalize<<<(L.n + 127) / 128, 128, 0, ctx->stream>>>(
        A, ctx->frames.as<int32_t>(),
        L.d_totals_final ? reinterpret_cast<const unsigned long long *>(L.d_totals_final) : tot,
        m->desc.gain[0], m->desc.gain[1],
        m->desc.gain[2], m->prob ? 1 : 0, (double)ne, L.d_xyz_out, L.d_gain_out,
        reinterpret_cast<unsigned long long *>(L.d_counts_out));
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_debug_trace(nbt_ctx ctx, nbt_map m, const int32_t *d_o, const int32_t *d_e, int32_t n_rays,
                              int32_t max_visits, int32_t *d_ijk, uint8_t *d_code, int32_t *d_len,
                              uint32_t *d_counts, bool wide)
{
    if (n_rays == 0) return NBT_OK;
    const DebugFn fn = kDebugFns[wide][m->layout == kLayoutMorton][store_kind(m)];
    fn<<<dim3((n_rays + 127) / 128), dim3(128), 0, ctx->stream>>>(view_of(m), d_o, d_e, n_rays, max_visits, d_ijk,
                                                                   d_code, d_len, d_counts);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

// The int32 decision terms are exact while every |E_a - O_a| < 2^30 - 1 (k_id.cu header).
bool debug_needs_wide(const int32_t *o_q16, const int32_t *e_q16, int32_t n_rays)
{
    for (int32_t i = 0; i < 3 * n_rays; ++i) {
        long long d = (long long)e_q16[i] - o_q16[i];
        if (d < 0) d = -d;
        if (d >= (1ll << 30) - 1) return true;
    }
    return false;
}

nbt_status launch_debug_frames(nbt_ctx ctx, nbt_map m, const double poi[3], const double *d_persp, int32_t n,
                               const nbt_camera &cam, double range, int32_t *d_frames)
{
    if (n == 0) return NBT_OK;
    FrameArgs A = frame_args(m, d_persp, 0, 1, n, poi, cam, range);
    k_debug_frames<<<(n + 127) / 128, 128, 0, ctx->stream>>>(A, d_frames);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
