// The exact integer 3D-DDA of the walk (reading Q13), shared by the
// ID trace (k_id.cu) and the map integration (k_integrate.cu).  See k_id.cu's header for
// the derivation of the int32 decision terms.
#pragma once

#include "nbt_internal.cuh"

namespace nbt {
namespace dda {

#ifndef NBT_DDA_PRED
#define NBT_DDA_PRED 1   // int32 step for the linear layout: 1 = predicated, "x first" from one LOP3 with a
                         // predicate output where the caller asks for it (the 2-bit store) and from two
                         // compares otherwise (the byte stores); 3 / 4 = LOP3 / two compares everywhere;
                         // 0 = the flag form (A/B builds)
#endif

constexpr int kQShift = 16;      // walk coordinates: Q16, the frames' lattice

struct MapView {
    const uint32_t *__restrict__ words;
    int nx, ny, nz;
    int px;          // linear layout: padded x extent
    int pxy;         // linear layout: padded x*y extent
    uint32_t mx, my, mz;   // Morton layout: bit masks of each axis (3 * pbits bits)
    int policy;      // NBT_OUTSIDE_UNKNOWN / NBT_OUTSIDE_CLIP
};

template <int L>
__device__ __forceinline__ uint32_t grid_index(const MapView &m, int x, int y, int z)
{
    if (L == kLayoutMorton)
        return (dilate3((uint32_t)x) | (dilate3((uint32_t)y) << 1) | (dilate3((uint32_t)z) << 2)) &
               (m.mx | m.my | m.mz);
    return (uint32_t)(x + kBorder) + (uint32_t)m.px * (uint32_t)(y + kBorder) +
           (uint32_t)m.pxy * (uint32_t)(z + kBorder);
}

// 2-bit store: the code of the voxel whose bit offset in the store is ib (= 2 x its index;
// the first voxel of a word sits at the top, map_store.cuh): rotate it to bits 30-31.
__device__ __forceinline__ uint32_t code_of(uint32_t word, uint32_t ib)
{
    return __funnelshift_l(word, word, ib) >> 30;      // shift amount taken mod 32
}

// Per-ray walk state.  T = int (rays < 2^14 voxels per axis, k_id.cu header) or long long.
template <typename T>
struct Walk {
    T qxy, qxz, qyz;           // sign decides the next axis (see header)
    T ax, ay, az;              // |D_a| in Q16 units
    T nax;                     // -|D_x| (hot path)
    uint32_t idx;              // linear: padded index of the current voxel (in-grid walk) << SH,
                               // SH = 1 for the 2-bit store (idx = the code's bit offset); Morton: address
    int dX, dY, ndZ;           // linear: idx increments of a step along x, y and (negated) z
    uint32_t rx, ry, rz;       // Morton: per-axis dilated coordinates in "decrement form"
    uint32_t xinv;             // Morton: bits to flip (axes walked in + direction)
    int s, n;                  // current step (0 = origin voxel) and total steps
    int s0;                    // step at which the walk entered the grid
    uint32_t nf;               // Free voxels counted so far in the grid
    uint32_t ng;               // 8-bit store: Eq. 2 gain counted so far (1/63 units)
    uint32_t pre;              // visits outside the grid before entering it
    int vx, vy, vz;            // voxel coordinates (entry path / debug only)
    int sx, sy, sz;            // +-1 per axis
};

template <typename T>
__device__ __forceinline__ void walk_setup(Walk<T> &w, const int o[3], const int e[3])
{
    // 32-bit operands throughout (|D| < 2^31: both ends inside (-2^30, 2^30); N in [0, 65536];
    // v << 16 in [-2^30, 2^30]), 64-bit only for the products N_a |D_b| < 2^47 (one 32x32->64
    // multiply-add each)
    uint32_t ad[3], N[3];
    int neg[3], v[3];
    int n = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int D = e[a] - o[a];
        neg[a] = D < 0;
        ad[a] = neg[a] ? (uint32_t)(-D) : (uint32_t)D;
        v[a] = o[a] >> kQShift;                  // floor
        const int ve = e[a] >> kQShift;
        n += (ve > v[a]) ? ve - v[a] : v[a] - ve;
        N[a] = neg[a] ? (uint32_t)(o[a] - (v[a] << kQShift))
                      : (uint32_t)(((v[a] + 1) << kQShift) - o[a]);   // in [0, 65536]
    }
    // tie favours the lower axis unless it moves negatively and the other positively
    const long long fxy = (long long)((unsigned long long)N[0] * ad[1]) - (long long)((unsigned long long)N[1] * ad[0]) -
                          ((neg[0] && !neg[1]) ? 0 : 1);
    const long long fxz = (long long)((unsigned long long)N[0] * ad[2]) - (long long)((unsigned long long)N[2] * ad[0]) -
                          ((neg[0] && !neg[2]) ? 0 : 1);
    const long long fyz = (long long)((unsigned long long)N[1] * ad[2]) - (long long)((unsigned long long)N[2] * ad[1]) -
                          ((neg[1] && !neg[2]) ? 0 : 1);
    w.qxy = (T)(fxy >> kQShift);                 // arithmetic shift = floor division by S
    w.qxz = (T)(fxz >> kQShift);
    w.qyz = (T)(fyz >> kQShift);
    w.ax = (T)ad[0]; w.ay = (T)ad[1]; w.az = (T)ad[2];
    w.nax = -w.ax;
    w.sx = neg[0] ? -1 : 1;
    w.sy = neg[1] ? -1 : 1;
    w.sz = neg[2] ? -1 : 1;
    w.vx = v[0]; w.vy = v[1]; w.vz = v[2];
    w.s = 0;
    w.n = n;
    w.nf = 0;
    w.ng = 0;
    w.pre = 0;
}

__device__ __forceinline__ int mad_i32(int a, int b, int c)
{
    int d;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// One DDA step: pick the axis, update the two decision terms that involve it, and move
// the map address.  Linear layout: idx += step of the axis.  Morton layout: every axis
// register holds its dilated coordinate so that a step is always a dilated DECREMENT
// (axes walked in + direction are stored complemented within their bits), i.e.
// r = (r - lsb) & mask, and the address is (rx | ry | rz) ^ xinv.
//
// Hot path (int32, no coordinates, linear layout): the axis choice as four predicates (4 ISETP,
// chained on the previous results; or 1 LOP3 with a predicate output + 2 ISETP, XLOP), the
// decision-term updates as 6 predicated adds and the new index as one add and two predicated
// overwrites -- 13 (12) instructions, none with more than two register sources, which ptxas
// spreads over the ALU (IADD3) and FMA (VIADD) pipes.  The register-only ceiling of this form is
// 2.23e12 visits/s against 1.92e12 for the earlier flag form (0/1 flags from the sign bits, 5 ALU
// ops and 9 multiply-adds by the flags: three register sources each), same decision terms
// (tools/dda_step_forms.cu, profiles/r02_s4_step_forms.log).  The Morton layout keeps the flag form.
// (Measured alternatives: 0/-1 masks with the negated magnitudes; one or two
// decision terms on the ALU pipe as AND + 3-input add, 4-14% slower.)
template <typename T, int L, bool COORDS, bool XLOP = false>
__device__ __forceinline__ void walk_step(Walk<T> &w, const MapView &m)
{
    if constexpr (sizeof(T) == 4 && !COORDS && L != kLayoutMorton && NBT_DDA_PRED) {
        constexpr bool lop = NBT_DDA_PRED == 3 || (NBT_DDA_PRED == 1 && XLOP);
        // x first: q_xy < 0 and q_xz < 0; y first: not x and q_yz < 0; z first: neither
        // the new index goes to a fresh register (the batch still reads the old one for its
        // rotate): one unconditional add and two predicated overwrites
        uint32_t nidx;
        if constexpr (!lop) {
            asm("{\n\t.reg .pred t, px, py, pz;\n\t"
            "setp.lt.s32 t, %1, 0;\n\t"
            "setp.lt.and.s32 px, %0, 0, t;\n\t"
            "setp.lt.and.s32 py, %2, 0, !px;\n\t"
            "setp.ge.and.s32 pz, %2, 0, !px;\n\t"
            "sub.s32 %3, %4, %10;\n\t"
            "@px add.s32 %0, %0, %5;\n\t"
            "@px add.s32 %1, %1, %6;\n\t"
            "@px add.s32 %3, %4, %8;\n\t"
            "@py sub.s32 %0, %0, %7;\n\t"
            "@py add.s32 %2, %2, %6;\n\t"
            "@py add.s32 %3, %4, %9;\n\t"
            "@pz sub.s32 %1, %1, %7;\n\t"
            "@pz sub.s32 %2, %2, %5;\n\t}"
            : "+r"(w.qxy), "+r"(w.qxz), "+r"(w.qyz), "=&r"(nidx)
            : "r"(w.idx), "r"(w.ay), "r"(w.az), "r"(w.ax), "r"(w.dX), "r"(w.dY), "r"(w.ndZ));
        } else {
            // x first from one LOP3 with a predicate output, (q_xy & q_xz & sign bit) != 0: one
            // instruction fewer on the ALU pipe (2-bit store: D -3.4%, B -3.5%; byte store: C'
            // +0.8%, profiles/r02_s4_addrlea.log)
            asm("{\n\t.reg .pred tru, px, py, pz;\n\t.reg .b32 t;\n\t"
            "setp.eq.u32 tru, 0, 0;\n\t"
            "lop3.and.b32 t|px, %0, %1, 0x80000000, 0x80, tru;\n\t"
            "setp.lt.and.s32 py, %2, 0, !px;\n\t"
            "setp.ge.and.s32 pz, %2, 0, !px;\n\t"
            "sub.s32 %3, %4, %10;\n\t"
            "@px add.s32 %0, %0, %5;\n\t"
            "@px add.s32 %1, %1, %6;\n\t"
            "@px add.s32 %3, %4, %8;\n\t"
            "@py sub.s32 %0, %0, %7;\n\t"
            "@py add.s32 %2, %2, %6;\n\t"
            "@py add.s32 %3, %4, %9;\n\t"
            "@pz sub.s32 %1, %1, %7;\n\t"
            "@pz sub.s32 %2, %2, %5;\n\t}"
            : "+r"(w.qxy), "+r"(w.qxz), "+r"(w.qyz), "=&r"(nidx)
            : "r"(w.idx), "r"(w.ay), "r"(w.az), "r"(w.ax), "r"(w.dX), "r"(w.dY), "r"(w.ndZ));
        }
        w.idx = nidx;
    } else if constexpr (sizeof(T) == 4 && !COORDS) {
        const int t1 = w.qxy & w.qxz;            // sign: x first
        const int t2 = w.qyz & ~t1;              // sign: y first
        const int px = (int)((unsigned)t1 >> 31);
        const int py = (int)((unsigned)t2 >> 31);
        const int npz = px + py - 1;             // -1 if z first, else 0
        w.qxy = mad_i32(px, w.ay, mad_i32(py, w.nax, w.qxy));
        w.qxz = mad_i32(px, w.az, mad_i32(npz, w.ax, w.qxz));
        w.qyz = mad_i32(py, w.az, mad_i32(npz, w.ay, w.qyz));
        if (L == kLayoutMorton) {
            w.rx = (uint32_t)mad_i32(px, -1, (int)w.rx) & m.mx;
            w.ry = (uint32_t)mad_i32(py, -2, (int)w.ry) & m.my;
            w.rz = (uint32_t)mad_i32(npz, 4, (int)w.rz) & m.mz;
            w.idx = (w.rx | w.ry | w.rz) ^ w.xinv;
        } else {
            w.idx = (uint32_t)mad_i32(px, w.dX, mad_i32(py, w.dY, mad_i32(npz, w.ndZ, (int)w.idx)));
        }
    } else {
        const bool px = (w.qxy & w.qxz) < 0;     // both negative
        const bool py = !px && w.qyz < 0;
        const bool pz = !px && !py;
        if (px) { w.qxy += w.ay; w.qxz += w.az; }
        if (py) { w.qxy -= w.ax; w.qyz += w.az; }
        if (pz) { w.qxz -= w.ax; w.qyz -= w.ay; }
        if (L == kLayoutMorton) {
            if (px) w.rx = (w.rx - 1u) & m.mx;
            if (py) w.ry = (w.ry - 2u) & m.my;
            if (pz) w.rz = (w.rz - 4u) & m.mz;
            w.idx = (w.rx | w.ry | w.rz) ^ w.xinv;
        } else {
            if (px) w.idx += w.dX;
            if (py) w.idx += w.dY;
            if (pz) w.idx -= w.ndZ;
        }
        if (COORDS) {
            if (px) w.vx += w.sx;
            if (py) w.vy += w.sy;
            if (pz) w.vz += w.sz;
        }
    }
}

__device__ __forceinline__ bool inside(const MapView &m, int x, int y, int z)
{
    return (unsigned)x < (unsigned)m.nx && (unsigned)y < (unsigned)m.ny && (unsigned)z < (unsigned)m.nz;
}

}  // namespace dda
}  // namespace nbt
