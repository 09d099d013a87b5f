"""Exact-rational brute-force voxel membership -- TEST INFRASTRUCTURE ONLY.

Independent of oracle.c (no event walk, no cross products): for a segment
P(t) = o + t d, t in [0, 1] (o, d rational, voxel units) it decides, voxel by
voxel over the bounding box, whether the closed segment meets the half-open
voxel [v, v+1)^3 (the map semantics O-1 of DESIGN.md) or the closed voxel
[v, v+1]^3, by intersecting per-axis parameter intervals with Fractions.  It
also lists the exact parameters at which two axes cross boundaries at the same
t in the same direction (edge/corner ties), where the 6-connected walk inserts
one voxel that no point of the segment lies in (reading Q13).
"""
from __future__ import annotations

from fractions import Fraction as Fr
from math import floor

Q = 65536   # the walk's fixed point: Q16 (reading Q19)


def _axis_interval(o, d, lo, hi, closed_cube):
    """Parameter set {t : lo <= o + t d < hi} (or <= hi if closed_cube) as
    (a, a_closed, b, b_closed), before clipping to [0, 1]; None if empty."""
    if d == 0:
        inside = (lo <= o <= hi) if closed_cube else (lo <= o < hi)
        return (Fr(-10**9), True, Fr(10**9), True) if inside else None
    ta, tb = (lo - o) / d, (hi - o) / d
    if d > 0:   # P increasing: lo reached at ta (closed), hi reached at tb
        return (ta, True, tb, closed_cube)
    # P decreasing: hi at tb (open unless closed cube), lo at ta (closed)
    return (tb, closed_cube, ta, True)


def _meets(o, d, v, closed_cube):
    a, a_c, b, b_c = Fr(0), True, Fr(1), True
    for k in range(3):
        iv = _axis_interval(o[k], d[k], Fr(v[k]), Fr(v[k] + 1), closed_cube)
        if iv is None:
            return False
        lo, lo_c, hi, hi_c = iv
        if lo > a or (lo == a and not lo_c):
            a, a_c = lo, lo_c
        if hi < b or (hi == b and not hi_c):
            b, b_c = hi, hi_c
    return a < b or (a == b and a_c and b_c)


def segment(o_q, e_q):
    o = [Fr(int(x), Q) for x in o_q]
    e = [Fr(int(x), Q) for x in e_q]
    return o, [e[k] - o[k] for k in range(3)]


def candidate_voxels(o, d):
    lo = [floor(min(o[k], o[k] + d[k])) - 1 for k in range(3)]
    hi = [floor(max(o[k], o[k] + d[k])) + 1 for k in range(3)]
    for x in range(lo[0], hi[0] + 1):
        for y in range(lo[1], hi[1] + 1):
            for z in range(lo[2], hi[2] + 1):
                yield (x, y, z)


def floor_set(o_q, e_q):
    """{floor(P(t)) : t in [0,1]} -- voxels containing a point of the closed segment."""
    o, d = segment(o_q, e_q)
    return {v for v in candidate_voxels(o, d) if _meets(o, d, v, closed_cube=False)}


def touch_set(o_q, e_q):
    """Voxels whose CLOSED cube meets the closed segment."""
    o, d = segment(o_q, e_q)
    return {v for v in candidate_voxels(o, d) if _meets(o, d, v, closed_cube=True)}


def _crossings(o, d):
    """Per axis: list of (t, sign) of the boundary crossings that change floor(P)."""
    out = []
    for k in range(3):
        ts = []
        if d[k] > 0:
            b = floor(o[k]) + 1
            while True:
                t = (b - o[k]) / d[k]
                if t > 1:
                    break
                ts.append(t); b += 1
        elif d[k] < 0:
            b = floor(o[k])
            while True:
                t = (o[k] - b) / (-d[k])
                if t >= 1:
                    break
                ts.append(t); b -= 1
        out.append(ts)
    return out


def same_sign_ties(o_q, e_q):
    """Exact parameters where two axes moving the same way cross at the same t."""
    o, d = segment(o_q, e_q)
    cr = _crossings(o, d)
    ties = []
    for a in range(3):
        for b in range(a + 1, 3):
            if d[a] == 0 or d[b] == 0 or (d[a] > 0) != (d[b] > 0):
                continue
            ties.extend(sorted(set(cr[a]) & set(cr[b])))
    return ties


def enter_param(o_q, e_q, v):
    """Smallest t at which P(t) lies in the half-open voxel v (None if never)."""
    o, d = segment(o_q, e_q)
    a, a_c, b, b_c = Fr(0), True, Fr(1), True
    for k in range(3):
        iv = _axis_interval(o[k], d[k], Fr(v[k]), Fr(v[k] + 1), False)
        if iv is None:
            return None
        lo, lo_c, hi, hi_c = iv
        if lo > a or (lo == a and not lo_c):
            a, a_c = lo, lo_c
        if hi < b or (hi == b and not hi_c):
            b, b_c = hi, hi_c
    if a < b or (a == b and a_c and b_c):
        return a
    return None
