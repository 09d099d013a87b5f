// Device-side addressing of the packed voxel-map store (layouts and value widths are
// described in k_map.cu's header), shared by the map kernels and the map integration.
#pragma once

#include "nbt_internal.cuh"

namespace nbt {

struct Geom {
    int layout;
    int vbits;                 // 2 or 8
    int prob;                  // 8-bit store holds the Eq. 2 gain in bits 2-7 (f1)
    int nx, ny, nz;
    uint32_t px, py;           // linear padded extents
    uint32_t def_level[3];     // 8-bit store: level used for U / F / O when none is given
};

// Store index of grid voxel (x, y, z).
__device__ __forceinline__ uint64_t store_index(const Geom &g, uint32_t x, uint32_t y, uint32_t z)
{
    if (g.layout == kLayoutMorton) return dilate3(x) | (dilate3(y) << 1) | (dilate3(z) << 2);
    return (uint64_t)(x + kBorder) + (uint64_t)g.px * ((uint64_t)(y + kBorder) + (uint64_t)g.py * (z + kBorder));
}

__device__ __forceinline__ uint32_t word_of(const Geom &g, uint64_t i) { return (uint32_t)(i >> (g.vbits == 2 ? 4 : 2)); }
__device__ __forceinline__ uint32_t shift_of(const Geom &g, uint64_t i)
{
    // 2-bit store: voxel i % 16 of a word at bits 31-2(i%16) .. 30-2(i%16) (first voxel at the
    // top, so the walk brings a code to bits 30-31 with one left rotate by its bit offset 2i)
    return g.vbits == 2 ? 30u - (uint32_t)(i & 15) * 2 : (uint32_t)(i & 3) * 8;
}

// The stored value of a grid voxel: the state, or state | Eq. 2 gain (1/63 units) << 2.
__device__ __forceinline__ uint32_t stored_value(const Geom &g, uint32_t code, uint32_t level)
{
    if (g.vbits == 2 || !g.prob) return code;
    const uint32_t gq = code == 0 ? 63u : (code == 1 ? level : 63u - level);
    return code | (gq << 2);
}

// Store geometry of a map handle (k_map.cu).
Geom geom_of(nbt_map m);

}  // namespace nbt
