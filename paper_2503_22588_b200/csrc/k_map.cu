// Voxel-map store kernels (8(f) row f1).
//
// Two layouts.  Linear (default): the nx*ny*nz grid is surrounded
// by a shell of kBorder sentinel voxels and stored x-fastest: voxel (x, y, z) is padded
// voxel (x+B, y+B, z+B) with index i = (x+B) + px*((y+B) + py*(z+B)), px = nx + 2B.
// Morton (NBT_MAP_LAYOUT=morton): a cube of side P = 2^pbits >= max(n) + 2 kBorder indexed
// by the bit-interleaved coordinates; every position outside the grid is sentinel.  The
// sentinel lets the walk detect leaving the grid with the same "code >= 2" test that
// detects an Occupied voxel, and its thickness keeps look-ahead loads inside the store.
//
// Two value widths.  2 bits per voxel (the three states, 0 U / 1 F / 2 O, 3 = sentinel),
// 16 voxels per word, the first at the top (bits 30-31): per-state gains (reading Q15).  8 bits per voxel (f1, exact Eq. 2,
// reading Q32), 4 voxels per word: bits 0-1 the state, bits 2-7 the voxel's Eq. 2 gain in
// units of 1/63 -- 63 for Unknown, level for Free (P = level/63), 63 - level for
// Occupied -- so the walk reads the gain with one shift.
#include <stdlib.h>

#include <cub/cub.cuh>

#include "nbt_internal.cuh"
#include "map_store.cuh"

namespace nbt {
namespace {

constexpr uint32_t kOutside = 3u;
// One thread per packed word.
__global__ void k_map_pack(const uint8_t *__restrict__ codes, const uint8_t *__restrict__ levels, Geom g,
                           uint64_t nvox_pad, size_t nwords, uint32_t *__restrict__ words, int *err)
{
    size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    const int per = g.vbits == 2 ? 16 : 4;
    uint64_t i0 = (uint64_t)w * per;
    uint32_t x = 0, y = 0, z = 0;
    if (g.layout == kLayoutLinear) {
        x = (uint32_t)(i0 % g.px);
        uint64_t r = i0 / g.px;
        y = (uint32_t)(r % g.py);
        z = (uint32_t)(r / g.py);
    }
    uint32_t out = 0;
    bool bad = false;
    for (int k = 0; k < per; ++k) {
        uint32_t v = kOutside;
        int gx, gy, gz;
        if (g.layout == kLayoutMorton) {
            const uint32_t i = (uint32_t)(i0 + k);
            gx = (int)compact3(i); gy = (int)compact3(i >> 1); gz = (int)compact3(i >> 2);
        } else {
            gx = (int)x - kBorder; gy = (int)y - kBorder; gz = (int)z - kBorder;
            if (++x == g.px) { x = 0; if (++y == g.py) { y = 0; ++z; } }
        }
        if (i0 + k < nvox_pad && gx >= 0 && gy >= 0 && gz >= 0 && gx < g.nx && gy < g.ny && gz < g.nz) {
            const size_t src = (size_t)gx + (size_t)g.nx * ((size_t)gy + (size_t)g.ny * gz);
            uint32_t c = codes[src];
            if (c > 2u) { bad = true; c = 0u; }
            uint32_t lv = levels ? levels[src] : g.def_level[c];
            if (lv > 63u) { bad = true; lv = 63u; }
            v = stored_value(g, c, lv);
        }
        out |= v << (g.vbits == 2 ? 30 - 2 * k : 8 * k);     // shift_of (map_store.cuh)
    }
    words[w] = out;
    if (bad) atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
}

// S:66-74 classification: unobserved -> U; P >= t_occ -> O; P <= t_free -> F; else U.  With
// levels_out (8-bit store): level = round-half-even(63 clamp(P, 0, 1)), 0 if unobserved (Q32).
__global__ void k_map_classify(const float *__restrict__ p, const uint8_t *__restrict__ obs, size_t n,
                               double t_occ, double t_free, uint8_t *__restrict__ codes,
                               uint8_t *__restrict__ levels_out)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = (double)p[i];
    uint8_t c = NBT_UNKNOWN;
    if (obs[i]) c = (v >= t_occ) ? NBT_OCCUPIED : (v <= t_free ? NBT_FREE : NBT_UNKNOWN);
    codes[i] = c;
    if (levels_out) {
        const double cl = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        levels_out[i] = obs[i] ? (uint8_t)__double2int_rn(__dmul_rn(cl, 63.0)) : 0;
    }
}

// Delta keys: (linear voxel index << pbits) | array position, in vbits + pbits bits (just
// enough for nx*ny*nz and n, so the radix sort runs only the passes it needs); invalid
// deltas get the all-ones key, which sorts last and no valid key reaches.
__global__ void k_delta_keys(const int32_t *__restrict__ ijk, const uint8_t *__restrict__ codes,
                             const uint8_t *__restrict__ levels, uint32_t n, int nx, int ny, int nz, int pbits,
                             unsigned long long bad, unsigned long long *__restrict__ keys, int *err)
{
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
    bool ok = x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz && codes[i] <= 2 &&
              (!levels || levels[i] <= 63);
    if (!ok) {
        keys[i] = bad;
        atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
        return;
    }
    unsigned long long lin = (unsigned long long)x + (unsigned long long)nx * ((unsigned long long)y +
                                                                             (unsigned long long)ny * z);
    keys[i] = (lin << pbits) | i;
}

// After sorting, the last key of each voxel run is the last delta in array order (Q30):
// only that one writes.  Distinct voxels may share a word, so the field is changed with
// one atomicXor; the thread's own field is never touched by another thread.
__global__ void k_delta_apply(const unsigned long long *__restrict__ keys, uint32_t n, int pbits,
                              unsigned long long bad, const int32_t *__restrict__ ijk,
                              const uint8_t *__restrict__ codes, const uint8_t *__restrict__ levels, Geom g,
                              uint32_t *words)
{
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long k = keys[i];
    if (k == bad) return;
    if (i + 1 < n && (keys[i + 1] >> pbits) == (k >> pbits)) return;
    uint32_t pos = (uint32_t)(k & ((1ull << pbits) - 1));
    uint64_t pi = store_index(g, (uint32_t)ijk[3 * pos], (uint32_t)ijk[3 * pos + 1], (uint32_t)ijk[3 * pos + 2]);
    uint32_t *w = words + word_of(g, pi);
    const uint32_t sh = shift_of(g, pi);
    const uint32_t mask = g.vbits == 2 ? 3u : 0xffu;
    const uint32_t c = codes[pos];
    const uint32_t nw = stored_value(g, c, levels ? levels[pos] : g.def_level[c]);
    const uint32_t old = (*(volatile uint32_t *)w >> sh) & mask;
    if (old != nw) atomicXor(w, (old ^ nw) << sh);
}

// Winner-array form of the delta update (no sort): every valid delta i raises its voxel's
// winner slot to i + 1 (atomicMax), so the slot ends at the LAST delta in array order (Q30);
// the winner then writes the field and clears the slot (a loser that reads the slot after
// the clear sees 0, never its own i + 1), leaving the array zeroed for the next update.
__global__ void k_delta_win(const int32_t *__restrict__ ijk, const uint8_t *__restrict__ codes,
                            const uint8_t *__restrict__ levels, uint32_t n, int nx, int ny, int nz, uint32_t *win,
                            int *err)
{
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
    const bool ok = x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz && codes[i] <= 2 &&
                    (!levels || levels[i] <= 63);
    if (!ok) {
        atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
        return;
    }
    const uint32_t lin = (uint32_t)x + (uint32_t)nx * ((uint32_t)y + (uint32_t)ny * (uint32_t)z);
    atomicMax(win + lin, i + 1u);
}

__global__ void k_delta_apply_win(const int32_t *__restrict__ ijk, const uint8_t *__restrict__ codes,
                                  const uint8_t *__restrict__ levels, uint32_t n, Geom g, uint32_t *win,
                                  uint32_t *words)
{
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
    if (x < 0 || y < 0 || z < 0 || x >= g.nx || y >= g.ny || z >= g.nz) return;
    const uint32_t lin = (uint32_t)x + (uint32_t)g.nx * ((uint32_t)y + (uint32_t)g.ny * (uint32_t)z);
    if (win[lin] != i + 1u) return;                     // a later delta of this voxel wins
    win[lin] = 0u;
    const uint64_t pi = store_index(g, (uint32_t)x, (uint32_t)y, (uint32_t)z);
    uint32_t *w = words + word_of(g, pi);
    const uint32_t sh = shift_of(g, pi);
    const uint32_t mask = g.vbits == 2 ? 3u : 0xffu;
    const uint32_t c = codes[i];
    const uint32_t nw = stored_value(g, c, levels ? levels[i] : g.def_level[c]);
    const uint32_t old = (*(volatile uint32_t *)w >> sh) & mask;
    if (old != nw) atomicXor(w, (old ^ nw) << sh);
}

// Small delta sets: both passes in one single-block launch, the block barrier between them
// (every atomicMax of the block is performed before any winner test reads the array).
constexpr int kDeltaOneBlock = 1024;
#ifndef NBT_DELTA_SMALL
#define NBT_DELTA_SMALL (8 * kDeltaOneBlock)     // largest delta set of the single-block form
#endif
__global__ void __launch_bounds__(kDeltaOneBlock)
    k_delta_win_apply_small(const int32_t *__restrict__ ijk, const uint8_t *__restrict__ codes,
                            const uint8_t *__restrict__ levels, uint32_t n, Geom g, uint32_t *win, uint32_t *words,
                            int *err)
{
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
        const bool ok = x >= 0 && y >= 0 && z >= 0 && x < g.nx && y < g.ny && z < g.nz && codes[i] <= 2 &&
                        (!levels || levels[i] <= 63);
        if (!ok) {
            atomicCAS(err, 0, (int)NBT_ERR_INVALID_ARG);
            continue;
        }
        atomicMax(win + ((uint32_t)x + (uint32_t)g.nx * ((uint32_t)y + (uint32_t)g.ny * (uint32_t)z)), i + 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
        if (x < 0 || y < 0 || z < 0 || x >= g.nx || y >= g.ny || z >= g.nz) continue;
        const uint32_t lin = (uint32_t)x + (uint32_t)g.nx * ((uint32_t)y + (uint32_t)g.ny * (uint32_t)z);
        if (*(volatile uint32_t *)(win + lin) != i + 1u) continue;     // a later delta of this voxel wins
        win[lin] = 0u;
        const uint64_t pi = store_index(g, (uint32_t)x, (uint32_t)y, (uint32_t)z);
        uint32_t *w = words + word_of(g, pi);
        const uint32_t sh = shift_of(g, pi);
        const uint32_t mask = g.vbits == 2 ? 3u : 0xffu;
        const uint32_t c = codes[i];
        const uint32_t nw = stored_value(g, c, levels ? levels[i] : g.def_level[c]);
        const uint32_t old = (*(volatile uint32_t *)w >> sh) & mask;
        if (old != nw) atomicXor(w, (old ^ nw) << sh);
    }
}

// Dense codes (and, for the 8-bit store, the probability levels) of the grid.
__global__ void k_map_unpack(const uint32_t *__restrict__ words, Geom g, uint8_t *__restrict__ codes,
                             uint8_t *__restrict__ levels)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t n = (size_t)g.nx * g.ny * g.nz;
    if (i >= n) return;
    uint32_t x = (uint32_t)(i % g.nx);
    size_t r = i / g.nx;
    uint32_t y = (uint32_t)(r % g.ny), z = (uint32_t)(r / g.ny);
    uint64_t pi = store_index(g, x, y, z);
    const uint32_t v = (words[word_of(g, pi)] >> shift_of(g, pi)) & (g.vbits == 2 ? 3u : 0xffu);
    const uint32_t c = v & 3u;
    if (codes) codes[i] = (uint8_t)c;
    if (levels) {
        const uint32_t gq = v >> 2;
        levels[i] = (uint8_t)(c == 1 ? gq : (c == 2 ? 63u - gq : 0u));
    }
}

inline unsigned blocks_for(size_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

Geom geom_of(nbt_map m)
{
    Geom g;
    g.layout = m->layout;
    g.vbits = m->vbits;
    g.prob = m->prob ? 1 : 0;
    g.nx = m->desc.nx; g.ny = m->desc.ny; g.nz = m->desc.nz;
    g.px = m->px; g.py = m->py;
    // a state-only write to the 8-bit store uses the per-state constants of the desc:
    // P_F = g_F and 1 - P_O = g_O (reading Q15), rounded to k/63
    g.def_level[0] = 0;
    g.def_level[1] = (uint32_t)nearbyint(fmin(fmax(m->desc.gain[1], 0.0), 1.0) * 63.0);
    g.def_level[2] = (uint32_t)nearbyint(fmin(fmax(1.0 - m->desc.gain[2], 0.0), 1.0) * 63.0);
    return g;
}

nbt_status launch_map_pack(nbt_ctx ctx, nbt_map m, const uint8_t *d_codes, const uint8_t *d_levels)
{
    if (m->nwords == 0) return NBT_OK;
    k_map_pack<<<blocks_for(m->nwords, 256), 256, 0, ctx->stream>>>(d_codes, d_levels, geom_of(m), m->nvox_pad,
                                                                     m->nwords, m->d_words, ctx->d_err);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_map_classify(nbt_ctx ctx, const float *d_p, const uint8_t *d_obs, size_t n, double t_occ,
                               double t_free, uint8_t *d_codes_out, uint8_t *d_levels_out)
{
    if (n == 0) return NBT_OK;
    k_map_classify<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(d_p, d_obs, n, t_occ, t_free, d_codes_out,
                                                                d_levels_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_map_update(nbt_ctx ctx, nbt_map m, const int32_t *d_ijk, const uint8_t *d_codes,
                             const uint8_t *d_levels, size_t n)
{
    if (n == 0) return NBT_OK;
    if (n >= (1ull << 31)) return fail(NBT_ERR_INVALID_ARG, "nbt_map_update: too many deltas");
    uint32_t nn = (uint32_t)n;
    ProfScope ps(ctx, NBT_KERNEL_MAP_UPDATE);
    nbt_status st;
    const uint64_t nvox = (uint64_t)m->desc.nx * m->desc.ny * m->desc.nz;
    // the winner array (4 B per voxel, zero between updates) is allocated on the first update
    // outside a graph capture; without it (or with NBT_OPT_DELTA_SORT) the sort form below is used
    const bool sort_form = ctx->opt.delta_sort != 0;
    if (!m->d_win && !g_capturing && !sort_form) {
        if (cudaMalloc(&m->d_win, nvox * 4) == cudaSuccess) {
            if (cudaMemsetAsync(m->d_win, 0, nvox * 4, ctx->stream) != cudaSuccess) {
                cudaFree(m->d_win);
                m->d_win = nullptr;
            }
        } else {
            m->d_win = nullptr;
            cudaGetLastError();
        }
    }
    if (m->d_win && !sort_form) {
        if (n <= NBT_DELTA_SMALL) {
            k_delta_win_apply_small<<<1, kDeltaOneBlock, 0, ctx->stream>>>(d_ijk, d_codes, d_levels, nn, geom_of(m),
                                                                          m->d_win, m->d_words, ctx->d_err);
            NBT_LAUNCHED(ctx);
            return NBT_OK;
        }
        k_delta_win<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(d_ijk, d_codes, d_levels, nn, m->desc.nx,
                                                                 m->desc.ny, m->desc.nz, m->d_win, ctx->d_err);
        NBT_LAUNCHED(ctx);
        k_delta_apply_win<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(d_ijk, d_codes, d_levels, nn, geom_of(m),
                                                                       m->d_win, m->d_words);
        NBT_LAUNCHED(ctx);
        return NBT_OK;
    }
    if ((st = ctx->keys.ensure(n * 8))) return st;
    if ((st = ctx->keys_alt.ensure(n * 8))) return st;
    auto *kin = ctx->keys.as<unsigned long long>();
    auto *kout = ctx->keys_alt.as<unsigned long long>();
    auto bits_for = [](unsigned long long v) { int b = 1; while (b < 64 && (v >> b)) ++b; return b; };
    const int pbits = bits_for(n - 1 > 0 ? n - 1 : 1);
    const int tbits = bits_for(nvox) + pbits;            // <= 33 + 31: always fits 64
    const unsigned long long bad = tbits >= 64 ? ~0ull : ((1ull << tbits) - 1);
    k_delta_keys<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(d_ijk, d_codes, d_levels, nn, m->desc.nx, m->desc.ny,
                                                              m->desc.nz, pbits, bad, kin, ctx->d_err);
    NBT_LAUNCHED(ctx);
    size_t tmp = 0;
    NBT_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kin, kout, (int)nn, 0, tbits, ctx->stream));
    if ((st = ctx->cub_tmp.ensure(tmp))) return st;
    NBT_CUDA(cub::DeviceRadixSort::SortKeys(ctx->cub_tmp.p, tmp, kin, kout, (int)nn, 0, tbits, ctx->stream));
    k_delta_apply<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(kout, nn, pbits, bad, d_ijk, d_codes, d_levels, geom_of(m),
                                                               m->d_words);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

nbt_status launch_map_unpack(nbt_ctx ctx, nbt_map m, uint8_t *d_codes_out, uint8_t *d_levels_out)
{
    size_t n = (size_t)m->desc.nx * m->desc.ny * m->desc.nz;
    k_map_unpack<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(m->d_words, geom_of(m), d_codes_out, d_levels_out);
    NBT_LAUNCHED(ctx);
    return NBT_OK;
}

}  // namespace nbt
