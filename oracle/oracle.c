/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the online local
 * Information Distribution (ID) of arxiv 2503.22588 (section III,
 * P:127-222) and of the IDW query of Eq. 4.  It exists to prove the
 * CUDA path right.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product library
 * (paper_2503_22588_b200/, libnbt.so) never links, includes or calls it, and the
 * two share no code, headers, tables or constants.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "Qn" = the reading numbered n in DESIGN.md (paper silent / ambiguous).
 * Everything is IEEE double, round-to-nearest, compiled with
 * -ffp-contract=off (no FMA contraction), so each written operation is
 * rounded exactly once.  Integer work uses int64 / __int128 so that no
 * overflow reasoning is needed to read it.
 *
 * Parity status per function:
 *   orc_trace_ray          pinned  (hand-traced rays, closed form, exact rational brute force)
 *   orc_frame_q16          pinned  (orthonormality, centre/corner rays, d_h worked examples)
 *   orc_id_compute         pinned  (SPEC worked examples, closed forms, invariants)
 *                          absolute g_P values on a real scene: "parity unpinned" (paper prints none, T25)
 *   orc_idw_query          pinned  (SPEC worked examples, convexity, H_NB identity)
 *   orc_idw_query_knn      pinned  (hand example, k >= N_P identity, k = 1 nearest, ties)
 *   orc_sample_perspectives pinned (forced-sample example, radius bounds, radial CDF)
 *   orc_classify           pinned  (S:69-74 threshold rule examples)
 *   orc_philox4x32         pinned  (published Random123 known-answer vectors)
 *   orc_voxel_filter       pinned  (S:53-56 examples, brute-force bucketing)
 *   orc_integrate          pinned  (S:61-64 examples, range truncation, hit-wins, exact touch sets)
 *   orc_occ_classify       pinned  (S:72-74 examples, round(63 sigmoid(L)) away from boundaries)
 *   orc_quantize_prob      pinned  (worked examples, hand-traced Eq. 2 ray, uniform-level identity)
 *   orc_map_update         pinned  (hand-worked last-wins example, rejection of bad deltas)
 *   orc_orientation_factor pinned  (SPEC worked examples, scale invariances)
 *   orc_info_cost          pinned  (closed forms)
 *   orc_eq1                pinned  (hand-computed forced samples)
 *   orc_camera_*           pinned  (s_G lattice counts of the SPEC / BASELINE examples)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_INVALID_ARG 1
#define ORC_ERR_DEGENERATE 2
#define ORC_ERR_EMPTY 3
#define ORC_ERR_SELFCHECK 9

#define QF 65536           /* frames, lattice and the walk: Q16, one voxel = 65536 units (Q19, SURVEY O-3/O-5) */
#define QLIM 1073741824LL  /* |coordinate| must stay below 2^30 in its unit (Q19) */

/* ------------------------------------------------------------------ map (O-1) */

typedef struct {
    int32_t nx, ny, nz;
    double voxel_size;       /* s_Vox */
    double origin[3];        /* world position of voxel (0,0,0)'s min corner */
    double gain[3];          /* g[U], g[F], g[O]  (Eq. 2, Q15) */
    int32_t outside_policy;  /* 0 = outside counts as Unknown, 1 = clip */
    const uint8_t *codes;    /* x fastest, nx*ny*nz */
    const uint8_t *levels;   /* NULL: per-state gains (Q15).  Else per-voxel probability
                                P = level / 63 (level 0..63) and Eq. 2 exactly (f1, Q32) */
} orc_map;

#define PLEVELS 63           /* P quantised to k / 63 (reading Q32) */

/* Eq. 2 for a quantised probability, in units of 1/63:
 * Unknown -> 1, Free -> P, Occupied -> 1 - P. */
static int64_t gain_q63(int code, int level)
{
    if (code == 0) return PLEVELS;
    if (code == 1) return level;
    return PLEVELS - level;
}

static int level_at(const orc_map *m, int64_t x, int64_t y, int64_t z)
{
    return m->levels[x + (int64_t)m->nx * (y + (int64_t)m->ny * z)];
}

/* code of voxel (x,y,z); -1 if outside the grid */
static int code_at(const orc_map *m, int64_t x, int64_t y, int64_t z)
{
    if (x < 0 || y < 0 || z < 0 || x >= m->nx || y >= m->ny || z >= m->nz) return -1;
    return m->codes[x + (int64_t)m->nx * (y + (int64_t)m->ny * z)];
}

/* ---------------------------------------------------------------- camera (a5) */

typedef struct {
    int32_t width, height;           /* ray lattice W x H */
    double fx, fy, cx, cy;           /* pinhole intrinsics in pixel units; 2cx = W-1, 2cy = H-1 */
    int32_t add_corners;             /* append the 4 far-plane corner rays */
    double tan_half_fov_h, tan_half_fov_v;
} orc_camera;

/* Corner-inclusive W x H lattice: pixel 0 and W-1 sit on the frustum borders
 * d_h = d_Cam tan(FoV_h/2), d_v = d_Cam tan(FoV_v/2). */
int orc_camera_from_fov(double fov_h, double fov_v, int32_t w, int32_t h, orc_camera *out)
{
    if (!out || w < 1 || h < 1 || !(fov_h > 0 && fov_h < M_PI) || !(fov_v > 0 && fov_v < M_PI))
        return ORC_ERR_INVALID_ARG;
    out->width = w;
    out->height = h;
    out->tan_half_fov_h = tan(fov_h / 2.0);
    out->tan_half_fov_v = tan(fov_v / 2.0);
    out->cx = (w - 1) / 2.0;
    out->cy = (h - 1) / 2.0;
    out->fx = (w > 1) ? (w - 1) / (2.0 * out->tan_half_fov_h) : 1.0;
    out->fy = (h > 1) ? (h - 1) / (2.0 * out->tan_half_fov_v) : 1.0;
    out->add_corners = 0;
    return ORC_OK;
}

/* The paper's s_G lattice (Q6-Q8): spacing s_G * s_Vox on the far
 * plane, centred on the axis, plus the 4 corner rays unless they coincide with
 * lattice points (Q9). */
int orc_camera_from_grid_scaling(double fov_h, double fov_v, double range, double voxel_size,
                                 double s_g, orc_camera *out)
{
    if (!out || !(range > 0) || !(voxel_size > 0) || !(s_g >= 1.0) ||
        !(fov_h > 0 && fov_h < M_PI) || !(fov_v > 0 && fov_v < M_PI))
        return ORC_ERR_INVALID_ARG;
    double delta = s_g * voxel_size;
    double th = tan(fov_h / 2.0), tv = tan(fov_v / 2.0);
    double d_h = range * th, d_v = range * tv;
    /* lattice offsets m*delta with |m*delta| <= d_h, judged with a 1e-9 relative
     * tolerance so that tan(pi/4) = 0.9999999999999999 still yields the border point */
    double rh = d_h / delta, rv = d_v / delta;
    double mh = floor(rh + 1e-9), mv = floor(rv + 1e-9);
    if (mh > 100000 || mv > 100000) return ORC_ERR_INVALID_ARG;
    out->width = 2 * (int32_t)mh + 1;
    out->height = 2 * (int32_t)mv + 1;
    out->cx = mh;
    out->cy = mv;
    out->fx = range / delta;
    out->fy = range / delta;
    out->tan_half_fov_h = th;
    out->tan_half_fov_v = tv;
    out->add_corners = !(fabs(rh - mh) <= 1e-9 && fabs(rv - mv) <= 1e-9);
    return ORC_OK;
}

int32_t orc_camera_num_rays(const orc_camera *cam)
{
    return cam->width * cam->height + (cam->add_corners ? 4 : 0);
}

/* -------------------------------------------------- frame + Q16 (a4, O-2, O-3) */

typedef struct {
    int32_t o[3];     /* origin p_P in Q16 voxel coordinates */
    int32_t a[3];     /* axis: (range/s) * fwd */
    int32_t rh[3];    /* half-pixel step along right */
    int32_t uh[3];    /* half-pixel step along up */
    int32_t rc[3];    /* corner offset along right (range/s * tan_h) */
    int32_t uc[3];    /* corner offset along up */
} orc_frame;

static int rne_q16(double v, int32_t *out)
{
    double q = v * 65536.0;                 /* exact: power of two */
    if (!(fabs(q) < (double)QLIM)) return ORC_ERR_INVALID_ARG;
    *out = (int32_t)nearbyint(q);           /* round half to even (default mode) */
    return ORC_OK;
}

/* Orientation: the view axis points from p_P to the PoI; roll fixed by
 * up-hint +z, fallback +x (Q4); far plane flat at d_Cam (Q5). */
int orc_frame_q16(const orc_map *m, const double poi[3], const double p[3], const orc_camera *cam,
                  double range, orc_frame *f, double fwd_out[3], double right_out[3], double up_out[3])
{
    double d[3] = {poi[0] - p[0], poi[1] - p[1], poi[2] - p[2]};
    if (d[0] == 0.0 && d[1] == 0.0 && d[2] == 0.0) return ORC_ERR_DEGENERATE;   /* Q18 */
    double n = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    double fwd[3] = {d[0] / n, d[1] / n, d[2] / n};
    double c[3] = {fwd[1], -fwd[0], 0.0};                      /* fwd x z */
    double nc = sqrt((c[0] * c[0] + c[1] * c[1]) + c[2] * c[2]);
    if (nc < 1e-6) {
        c[0] = 0.0; c[1] = fwd[2]; c[2] = -fwd[1];              /* fwd x x */
        nc = sqrt((c[0] * c[0] + c[1] * c[1]) + c[2] * c[2]);
    }
    double right[3] = {c[0] / nc, c[1] / nc, c[2] / nc};
    double up[3] = {right[1] * fwd[2] - right[2] * fwd[1],
                    right[2] * fwd[0] - right[0] * fwd[2],
                    right[0] * fwd[1] - right[1] * fwd[0]};
    double s = m->voxel_size;
    double rs = range / s;
    double hx = rs / (2.0 * cam->fx);
    double hy = rs / (2.0 * cam->fy);
    double ch = rs * cam->tan_half_fov_h;
    double cv = rs * cam->tan_half_fov_v;
    int st = ORC_OK;
    for (int k = 0; k < 3; ++k) {
        st |= rne_q16((p[k] - m->origin[k]) / s, &f->o[k]);
        st |= rne_q16(rs * fwd[k], &f->a[k]);
        st |= rne_q16(hx * right[k], &f->rh[k]);
        st |= rne_q16(hy * up[k], &f->uh[k]);
        st |= rne_q16(ch * right[k], &f->rc[k]);
        st |= rne_q16(cv * up[k], &f->uc[k]);
    }
    if (fwd_out) memcpy(fwd_out, fwd, sizeof fwd);
    if (right_out) memcpy(right_out, right, sizeof right);
    if (up_out) memcpy(up_out, up, sizeof up);
    return st ? ORC_ERR_INVALID_ARG : ORC_OK;
}

/* Endpoint of ray k (O-4): k runs row-major over (row kk, column i); corner rays
 * follow in the order (-,-), (+,-), (-,+), (+,+).  Returns INVALID_ARG if any
 * coordinate leaves (-2^30, 2^30). */
static int ray_endpoint(const orc_frame *f, const orc_camera *cam, int32_t k, int32_t e[3])
{
    int64_t v[3];
    int32_t nlat = cam->width * cam->height;
    if (k < nlat) {
        int64_t i = k % cam->width, kk = k / cam->width;
        int64_t mi = 2 * i - (cam->width - 1), mk = 2 * kk - (cam->height - 1);
        for (int c = 0; c < 3; ++c)
            v[c] = (int64_t)f->o[c] + f->a[c] + mi * f->rh[c] + mk * f->uh[c];
    } else {
        int32_t q = k - nlat;
        int64_t sr = (q & 1) ? 1 : -1, su = (q & 2) ? 1 : -1;
        for (int c = 0; c < 3; ++c)
            v[c] = (int64_t)f->o[c] + f->a[c] + sr * f->rc[c] + su * f->uc[c];
    }
    for (int c = 0; c < 3; ++c) {
        if (v[c] <= -QLIM || v[c] >= QLIM) return ORC_ERR_INVALID_ARG;
        e[c] = (int32_t)v[c];
    }
    return ORC_OK;
}

/* ------------------------------------------------------ exact DDA (a6, O-5, Q13) */

typedef struct {
    int64_t n_u, n_f, n_o;   /* per-state counts of the N_O counted voxels (Eq. 2) */
    int64_t lookups;         /* in-grid visits (memory-touching subset) */
    int64_t visits;          /* voxels visited including uncounted (clipped) ones */
    int64_t g63;             /* per-voxel-probability mode: 63 * g_R as an integer */
    double g;                /* g_R = sum of g(v_i) over the counted voxels, in visit order */
    int32_t stop;            /* 0 = reached the endpoint voxel, 1 = stopped on Occupied */
} orc_ray;

static int64_t floor_div(int64_t a, int64_t b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

/*
 * Walk the voxels of the segment O -> E (Q16 voxel coordinates: 65536 units per voxel,
 * SURVEY 8(c) O-5 with S = 65536).
 *
 * Definition followed: the point P(t) = O + t (E - O), t in [0,1], lies in voxel
 * floor(P(t)) (half-open voxels, O-1).  Moving in +a the index changes AT the
 * boundary parameter; moving in -a it changes just AFTER it.  Events are
 * therefore ordered by (t, positive-before-negative, axis x<y<z); same-sign
 * simultaneous crossings (edges/corners) are taken one axis at a time in axis
 * order, which keeps the path 6-connected (Q13).  The walk visits exactly
 * 1 + sum_a |floor(E_a) - floor(O_a)| voxels when it does not stop early.
 *
 * Each visited voxel is scored by its state (Eq. 2): outside the
 * grid is Unknown (Q14) unless the clip policy is set; the walk stops
 * after the first Occupied voxel, which is counted (Q11); the origin
 * voxel is counted (reading Q12).  If ijk_out != NULL the visited voxels (up to
 * max_visits) are written there and their codes (0/1/2, 255 = outside) to
 * code_out.
 */
int orc_trace_ray(const orc_map *m, const int32_t o[3], const int32_t e[3], int32_t max_visits,
                  int32_t *ijk_out, uint8_t *code_out, int32_t *len_out, orc_ray *r)
{
    int64_t v[3], ve[3], D[3], N[3];
    int neg[3];
    int64_t nsteps = 0;
    for (int a = 0; a < 3; ++a) {
        if (o[a] <= -QLIM || o[a] >= QLIM || e[a] <= -QLIM || e[a] >= QLIM) return ORC_ERR_INVALID_ARG;
        v[a] = floor_div(o[a], QF);
        ve[a] = floor_div(e[a], QF);
        D[a] = (int64_t)e[a] - o[a];
        neg[a] = D[a] < 0;
        /* distance (in Q16 units) from O to the next boundary crossed along a */
        N[a] = neg[a] ? (int64_t)o[a] - v[a] * QF : (v[a] + 1) * QF - o[a];
        nsteps += llabs(ve[a] - v[a]);
    }
    memset(r, 0, sizeof *r);
    int32_t len = 0;
    for (int64_t s = 0;; ++s) {
        /* visit v */
        int code = code_at(m, v[0], v[1], v[2]);
        if (ijk_out && len < max_visits) {
            ijk_out[3 * len + 0] = (int32_t)v[0];
            ijk_out[3 * len + 1] = (int32_t)v[1];
            ijk_out[3 * len + 2] = (int32_t)v[2];
            code_out[len] = (code < 0) ? 255 : (uint8_t)code;
        }
        ++len;
        r->visits++;
        if (code >= 0) r->lookups++;
        if (code < 0 && m->outside_policy == 1) {
            /* clipped: not counted */
        } else {
            int c = code < 0 ? 0 : code;
            if (m->levels) {
                int lv = code < 0 ? 0 : level_at(m, v[0], v[1], v[2]);
                int64_t gq = gain_q63(c, lv);
                r->g63 += gq;
                r->g += (c == 0) ? 1.0 : (c == 1 ? (double)lv / PLEVELS : 1.0 - (double)lv / PLEVELS);
            } else {
                r->g += m->gain[c];
            }
            if (c == 0) r->n_u++;
            else if (c == 1) r->n_f++;
            else { r->n_o++; r->stop = 1; break; }
        }
        if (s == nsteps) break;
        /* next event: active axis with the smallest (N_a/|D_a|, neg_a, a) */
        int best = -1;
        for (int a = 0; a < 3; ++a) {
            if (D[a] == 0) continue;
            if (best < 0) { best = a; continue; }
            __int128 lhs = (__int128)N[a] * (D[best] < 0 ? -D[best] : D[best]);
            __int128 rhs = (__int128)N[best] * (D[a] < 0 ? -D[a] : D[a]);
            if (lhs < rhs || (lhs == rhs && neg[a] < neg[best])) best = a;
        }
        v[best] += neg[best] ? -1 : 1;
        N[best] += QF;
    }
    if (len_out) *len_out = len;
    return ORC_OK;
}

/* The segment the walk follows for ray k: the perspective origin O and the ray's
 * far-plane endpoint E, both on the Q16 lattice (O-3, O-4; Q19). */
static int ray_segment_q16(const orc_frame *f, const orc_camera *cam, int32_t k, int32_t o16[3], int32_t e16[3])
{
    int st = ray_endpoint(f, cam, k, e16);
    if (st) return st;
    for (int c = 0; c < 3; ++c) o16[c] = f->o[c];
    return ORC_OK;
}

/* ---------------------------------------------- ID per perspective (a7, a8, O-6) */

typedef struct {
    double xyz[3];
    double gain;                  /* g_P,j */
    int64_t t_u, t_f, t_o, lookups;
    int64_t t_g;                  /* per-voxel-probability mode: 63 * sum of g_R */
} orc_persp_out;

/* g_P,j for perspective j = (1/N_E) sum_k g_R,k,j with
 * g_R,k,j = sum over the N_O counted voxels of g(v_i) (Eq. 2).
 * Canonical form (Q26): ((T_U g_U + T_F g_F) + T_O g_O) / N_E from integer
 * per-state totals.  The direct ray-order sum is also computed and must agree
 * (self-check of the two readings of P:214, Q26) within the worst-case bound of
 * recursive summation of nonnegative terms: T terms (every counted visit plus the N_E
 * per-ray sums) each rounded once, and each per-voxel term g(v) itself rounded once in
 * the probability mode, give |direct - exact| <= gamma_{2T} * exact, gamma_n =
 * n u / (1 - n u), u = 2^-53 (Higham, Accuracy and Stability, 4.2); the canonical form
 * adds at most gamma_8. */
static int one_perspective(const orc_map *m, const double poi[3], const double p[3],
                           const orc_camera *cam, double range, orc_persp_out *out)
{
    orc_frame f;
    int st = orc_frame_q16(m, poi, p, cam, range, &f, NULL, NULL, NULL);
    if (st) return st;
    int32_t ne = orc_camera_num_rays(cam);
    int64_t tu = 0, tf = 0, to = 0, tl = 0, tg = 0, nvis = 0;
    double direct = 0.0;
    for (int32_t k = 0; k < ne; ++k) {
        int32_t o[3], e[3];
        if ((st = ray_segment_q16(&f, cam, k, o, e))) return st;
        orc_ray r;
        if ((st = orc_trace_ray(m, o, e, 0, NULL, NULL, NULL, &r))) return st;
        direct += r.g;
        tu += r.n_u; tf += r.n_f; to += r.n_o; tl += r.lookups; tg += r.g63;
        nvis += r.n_u + r.n_f + r.n_o;
    }
    double canon = m->levels ? (double)tg / ((double)PLEVELS * (double)ne)
                             : (((double)tu * m->gain[0] + (double)tf * m->gain[1]) + (double)to * m->gain[2]) /
                                   (double)ne;
    direct = direct / (double)ne;
    const double u = ldexp(1.0, -53);
    const double nt = 2.0 * (double)(nvis + ne) + 8.0;
    const double gamma = nt * u / (1.0 - nt * u);
    double scale = fabs(canon) > fabs(direct) ? fabs(canon) : fabs(direct);
    if (fabs(direct - canon) > gamma * scale) return ORC_ERR_SELFCHECK;
    memcpy(out->xyz, p, 3 * sizeof(double));
    out->gain = canon;
    out->t_u = tu; out->t_f = tf; out->t_o = to; out->lookups = tl; out->t_g = tg;
    return ORC_OK;
}

/* The whole ID: every perspective j of the set, in input order (O-7).
 * Perspectives are independent; nthreads > 1 only spreads them over host
 * cores (each perspective is still evaluated by the same sequential loop).
 * Returns the first failing perspective's index in *bad_index. */
int orc_id_compute(const orc_map *m, const double poi[3], const double *persp, int32_t n_persp,
                   const orc_camera *cam, double range, int32_t nthreads,
                   double *xyz_out, double *gain_out, int64_t *counts_out, int64_t *tg_out, int32_t *bad_index)
{
    if (!m || !poi || !persp || !cam || n_persp < 0 || !(range > 0)) return ORC_ERR_INVALID_ARG;
    if (cam->width < 1 || cam->height < 1) return ORC_ERR_INVALID_ARG;
    int status = ORC_OK;
    int32_t bad = -1;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int32_t j = 0; j < n_persp; ++j) {
        orc_persp_out o;
        int st = one_perspective(m, poi, persp + 3 * (int64_t)j, cam, range, &o);
        if (st) {
#ifdef _OPENMP
#pragma omp critical
#endif
            {
                if (bad < 0 || j < bad) { bad = j; status = st; }
            }
            continue;
        }
        if (xyz_out) memcpy(xyz_out + 3 * (int64_t)j, o.xyz, 3 * sizeof(double));
        if (gain_out) gain_out[j] = o.gain;
        if (counts_out) {
            counts_out[4 * (int64_t)j + 0] = o.t_u;
            counts_out[4 * (int64_t)j + 1] = o.t_f;
            counts_out[4 * (int64_t)j + 2] = o.t_o;
            counts_out[4 * (int64_t)j + 3] = o.lookups;
        }
        if (tg_out) tg_out[j] = o.t_g;
    }
    if (bad_index) *bad_index = bad;
    return status;
}

/* Rays of one perspective, for per-ray parity: the Q16 segment ends (the origin is
 * common to all rays) and per-ray counts. */
int orc_perspective_rays(const orc_map *m, const double poi[3], const double p[3],
                         const orc_camera *cam, double range, int32_t *o_out, int32_t *e_out,
                         int64_t *ray_counts_out /* ne x 5: U,F,O,lookups,stop */)
{
    orc_frame f;
    int st = orc_frame_q16(m, poi, p, cam, range, &f, NULL, NULL, NULL);
    if (st) return st;
    int32_t ne = orc_camera_num_rays(cam);
    for (int32_t k = 0; k < ne; ++k) {
        int32_t o[3], e[3];
        if ((st = ray_segment_q16(&f, cam, k, o, e))) return st;
        if (o_out && k == 0) memcpy(o_out, o, sizeof o);
        if (e_out) memcpy(e_out + 3 * (int64_t)k, e, sizeof e);
        if (ray_counts_out) {
            orc_ray r;
            if ((st = orc_trace_ray(m, o, e, 0, NULL, NULL, NULL, &r))) return st;
            int64_t *rc = ray_counts_out + 5 * (int64_t)k;
            rc[0] = r.n_u; rc[1] = r.n_f; rc[2] = r.n_o; rc[3] = r.lookups; rc[4] = r.stop;
        }
    }
    return ORC_OK;
}

/* Frame export for tests: o,a,rh,uh,rc,uc (18 int32) and fwd,right,up (9 doubles). */
int orc_frame_export(const orc_map *m, const double poi[3], const double p[3], const orc_camera *cam,
                     double range, int32_t *q16_out, double *axes_out)
{
    orc_frame f;
    int st = orc_frame_q16(m, poi, p, cam, range, &f, axes_out, axes_out ? axes_out + 3 : NULL,
                           axes_out ? axes_out + 6 : NULL);
    if (st) return st;
    if (q16_out) memcpy(q16_out, &f, sizeof f);
    return ORC_OK;
}

/* ----------------------------------------------------- IDW query (a9, Eq. 4, O-8) */

/* G(x) = sum_u w_u * v_u(x),  v_u = sum_j g_j d_j^-p / sum_j d_j^-p,
 * over buffer entries u = 0 (oldest) .. m-1 (newest); w_u = 1/(m-u) so the
 * newest entry weighs 1 (Q21); with a full buffer m = N_B this is the
 * paper's 1/(N_B - u).  If a perspective is closer than zero_eps, v_u is the
 * gain of the nearest one (lowest j among ties) (Q23).  Sums over all
 * perspectives of the entry (Q22).  normalize != 0 divides by sum_u w_u. */
int orc_idw_query(int32_t n_entries, const int32_t *entry_sizes, const double *const *entry_xyz,
                  const double *const *entry_gain, const double *query_xyz, int32_t n_q,
                  double power_p, double zero_eps, int32_t normalize, double *g_out)
{
    if (n_entries <= 0) return ORC_ERR_EMPTY;
    for (int32_t e = 0; e < n_entries; ++e)
        if (entry_sizes[e] <= 0) return ORC_ERR_INVALID_ARG;
    for (int32_t q = 0; q < n_q; ++q) {
        const double *x = query_xyz + 3 * (int64_t)q;
        double g = 0.0, wsum = 0.0;
        for (int32_t e = 0; e < n_entries; ++e) {
            const double *P = entry_xyz[e];
            const double *G = entry_gain[e];
            int32_t np = entry_sizes[e];
            int32_t nearest = -1;
            double dmin = 0.0;
            double num = 0.0, den = 0.0;
            for (int32_t j = 0; j < np; ++j) {
                double dx = x[0] - P[3 * j], dy = x[1] - P[3 * j + 1], dz = x[2] - P[3 * j + 2];
                double d2 = (dx * dx + dy * dy) + dz * dz;
                double d = sqrt(d2);
                if (nearest < 0 || d < dmin) { nearest = j; dmin = d; }
                double w = (power_p == 2.0) ? 1.0 / d2 : pow(d2, -power_p / 2.0);
                num += G[j] * w;
                den += w;
            }
            double v = (dmin < zero_eps) ? G[nearest] : num / den;
            double wu = 1.0 / (double)(n_entries - e);
            g += wu * v;
            wsum += wu;
        }
        g_out[q] = normalize ? g / wsum : g;
    }
    return ORC_OK;
}

/* Optional k-nearest variant of Eq. 4 (reading Q22): "interpolates ...
 * across the nearest perspectives" read as the knn nearest ones of each entry,
 * nearest by squared distance with ties to the lower index; v_u sums them in ascending j.
 * knn >= the entry size gives orc_idw_query exactly.  The zero-distance rule is the same
 * as orc_idw_query's (nearest by d over the whole entry). */
typedef struct { double d2; int32_t j; } orc_dj;

static int dj_cmp(const void *a, const void *b)
{
    const orc_dj *x = (const orc_dj *)a, *y = (const orc_dj *)b;
    if (x->d2 != y->d2) return x->d2 < y->d2 ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

static int j_cmp(const void *a, const void *b)
{
    const orc_dj *x = (const orc_dj *)a, *y = (const orc_dj *)b;
    return (x->j > y->j) - (x->j < y->j);
}

int orc_idw_query_knn(int32_t n_entries, const int32_t *entry_sizes, const double *const *entry_xyz,
                      const double *const *entry_gain, const double *query_xyz, int32_t n_q, double power_p,
                      double zero_eps, int32_t normalize, int32_t knn, double *g_out)
{
    if (n_entries <= 0) return ORC_ERR_EMPTY;
    if (knn < 1) return ORC_ERR_INVALID_ARG;
    int32_t maxn = 0;
    for (int32_t e = 0; e < n_entries; ++e) {
        if (entry_sizes[e] <= 0) return ORC_ERR_INVALID_ARG;
        if (entry_sizes[e] > maxn) maxn = entry_sizes[e];
    }
    orc_dj *dj = (orc_dj *)malloc((size_t)maxn * sizeof *dj);
    if (!dj) return ORC_ERR_INVALID_ARG;
    for (int32_t q = 0; q < n_q; ++q) {
        const double *x = query_xyz + 3 * (int64_t)q;
        double g = 0.0, wsum = 0.0;
        for (int32_t e = 0; e < n_entries; ++e) {
            const double *P = entry_xyz[e];
            const double *G = entry_gain[e];
            int32_t np = entry_sizes[e];
            int32_t nearest = -1;
            double dmin = 0.0;
            for (int32_t j = 0; j < np; ++j) {
                double dx = x[0] - P[3 * j], dy = x[1] - P[3 * j + 1], dz = x[2] - P[3 * j + 2];
                dj[j].d2 = (dx * dx + dy * dy) + dz * dz;
                dj[j].j = j;
                double d = sqrt(dj[j].d2);
                if (nearest < 0 || d < dmin) { nearest = j; dmin = d; }
            }
            int32_t k = knn < np ? knn : np;
            qsort(dj, (size_t)np, sizeof *dj, dj_cmp);       /* the k nearest come first */
            qsort(dj, (size_t)k, sizeof *dj, j_cmp);         /* ... summed in ascending j */
            double num = 0.0, den = 0.0;
            for (int32_t t = 0; t < k; ++t) {
                double w = (power_p == 2.0) ? 1.0 / dj[t].d2 : pow(dj[t].d2, -power_p / 2.0);
                num += G[dj[t].j] * w;
                den += w;
            }
            double v = (dmin < zero_eps) ? G[nearest] : num / den;
            double wu = 1.0 / (double)(n_entries - e);
            g += wu * v;
            wsum += wu;
        }
        g_out[q] = normalize ? g / wsum : g;
    }
    free(dj);
    return ORC_OK;
}

/* ------------------------- orientation factor and information cost (f2) */

/* O(x): the cosine of the angle between the camera's actual optical axis and
 * the ideal orientation towards the PoI; 0 when the PoI is outside the field of view,
 * read as theta > theta_cut with theta_cut = min(FoV_h, FoV_v)/2.  The
 * test theta <= theta_cut is written as cos(theta) >= cos(theta_cut) (reading Q31).
 * Returns ORC_ERR_DEGENERATE if the position is within 1e-9 of the PoI. */
int orc_orientation_factor(const double pos[3], const double axis[3], const double poi[3], double cos_cut,
                           double *o_out)
{
    double d[3] = {poi[0] - pos[0], poi[1] - pos[1], poi[2] - pos[2]};
    double nd = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    if (nd < 1e-9) return ORC_ERR_DEGENERATE;
    double na = sqrt((axis[0] * axis[0] + axis[1] * axis[1]) + axis[2] * axis[2]);
    if (!(na > 0)) return ORC_ERR_INVALID_ARG;
    double c = ((axis[0] * d[0] + axis[1] * d[1]) + axis[2] * d[2]) / (na * nd);
    *o_out = (c >= cos_cut) ? c : 0.0;
    return ORC_OK;
}

/* c_I(x_{0:K}) = sum_k w_I / (O(x_k) G(x_k) + eps)  (eps = 1e-7 P:259) for each of
 * n_traj trajectories of `per` poses (K + 1 = per), poses in order; G by orc_idw_query. */
int orc_info_cost(int32_t n_entries, const int32_t *entry_sizes, const double *const *entry_xyz,
                  const double *const *entry_gain, const double *pos, const double *axis, int32_t n_traj,
                  int32_t per, const double poi[3], double cos_cut, double w_i, double eps, double power_p,
                  double zero_eps, int32_t normalize, double *o_out, double *g_out, double *c_out)
{
    int32_t n = n_traj * per;
    int st = orc_idw_query(n_entries, entry_sizes, entry_xyz, entry_gain, pos, n, power_p, zero_eps, normalize,
                           g_out);
    if (st) return st;
    for (int32_t t = 0; t < n_traj; ++t) {
        double c = 0.0;
        for (int32_t k = 0; k < per; ++k) {
            int32_t i = t * per + k;
            double o;
            if ((st = orc_orientation_factor(pos + 3 * (int64_t)i, axis + 3 * (int64_t)i, poi, cos_cut, &o)))
                return st;
            if (o_out) o_out[i] = o;
            c += w_i / (o * g_out[i] + eps);
        }
        c_out[t] = c;
    }
    return ORC_OK;
}

/* ------------------------------------------------ sampler (a3, Eq. 1, O-9, Q1-Q3) */

/* Philox4x32-10 (Salmon et al., Random123): counter-based, so the same draws
 * can be reproduced anywhere from (seed, counter). */
void orc_philox4x32(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static double u01(uint32_t b) { return ((double)b + 0.5) * (1.0 / 4294967296.0); }

/* p_P = p_POI + r_S X_R^{1/3} X / ||X||  (Eq. 1, P:149-151 with the PoI offset, Q2),
 * X ~ N(0, I_3) by Box-Muller (Muller's method), X_R ~ U(0,1) (Q1);
 * mode 1 ("surface") uses X_R = 1 (Q3).  Draw j, attempt a uses Philox counters
 * (j, a, 0, 0) for the normals and (j, a, 1, 0) for X_R; ||X|| < 1e-12 is
 * resampled with a+1. */
int orc_sample_perspectives(const double poi[3], double r_s, int32_t n, uint64_t seed, int32_t mode,
                            double *xyz_out)
{
    if (!poi || !xyz_out || n < 0 || !(r_s > 0) || (mode != 0 && mode != 1)) return ORC_ERR_INVALID_ARG;
    const double two_pi = 6.283185307179586;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int32_t j = 0; j < n; ++j) {
        for (uint32_t attempt = 0;; ++attempt) {
            uint32_t c0[4] = {(uint32_t)j, attempt, 0u, 0u}, b[4];
            orc_philox4x32(c0, key, b);
            double u0 = u01(b[0]), u1 = u01(b[1]), u2 = u01(b[2]), u3 = u01(b[3]);
            double r01 = sqrt(-2.0 * log(u0)), r23 = sqrt(-2.0 * log(u2));
            double X[3] = {r01 * cos(two_pi * u1), r01 * sin(two_pi * u1), r23 * cos(two_pi * u3)};
            double nx = sqrt((X[0] * X[0] + X[1] * X[1]) + X[2] * X[2]);
            if (nx < 1e-12) continue;
            double xr = 1.0;
            if (mode == 0) {
                uint32_t c1[4] = {(uint32_t)j, attempt, 1u, 0u}, b1[4];
                orc_philox4x32(c1, key, b1);
                xr = u01(b1[0]);
            }
            double scale = r_s * cbrt(xr);
            for (int k = 0; k < 3; ++k) xyz_out[3 * (int64_t)j + k] = poi[k] + scale * (X[k] / nx);
            break;
        }
    }
    return ORC_OK;
}

/* The Eq. 1 map applied to given draws (forced-sample pins). */
void orc_eq1(const double poi[3], double r_s, const double X[3], double x_r, double out[3])
{
    double nx = sqrt((X[0] * X[0] + X[1] * X[1]) + X[2] * X[2]);
    double scale = r_s * cbrt(x_r);
    for (int k = 0; k < 3; ++k) out[k] = poi[k] + scale * (X[k] / nx);
}

/* ------------------------------------------------- classification (Q16) */

/* Per-voxel probability for the exact Eq. 2 (f1): state by the rule below, and
 * level = round-half-even(clamp(P, 0, 1) * 63) (reading Q32); unobserved -> level 0. */
void orc_quantize_prob(const float *p, const uint8_t *observed, int64_t n, double t_occ, double t_free,
                       uint8_t *codes_out, uint8_t *levels_out)
{
    for (int64_t i = 0; i < n; ++i) {
        double v = (double)p[i];
        int c = 0;
        if (observed[i]) c = (v >= t_occ) ? 2 : (v <= t_free ? 1 : 0);
        codes_out[i] = (uint8_t)c;
        double cl = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        levels_out[i] = observed[i] ? (uint8_t)nearbyint(cl * PLEVELS) : 0;
    }
}

/* unobserved -> Unknown; P >= t_occ -> Occupied; P <= t_free -> Free; else Unknown. */
void orc_classify(const float *p, const uint8_t *observed, int64_t n, double t_occ, double t_free,
                  uint8_t *codes_out)
{
    for (int64_t i = 0; i < n; ++i) {
        if (!observed[i]) codes_out[i] = 0;
        else if ((double)p[i] >= t_occ) codes_out[i] = 2;
        else if ((double)p[i] <= t_free) codes_out[i] = 1;
        else codes_out[i] = 0;
    }
}

/* Map deltas (row a2): applied in array order, so the last delta of a voxel wins (Q30). */
int orc_map_update(uint8_t *codes, int32_t nx, int32_t ny, int32_t nz, const int32_t *ijk, const uint8_t *vals,
                   int64_t n)
{
    for (int64_t i = 0; i < n; ++i) {
        int64_t x = ijk[3 * i], y = ijk[3 * i + 1], z = ijk[3 * i + 2];
        if (x < 0 || y < 0 || z < 0 || x >= nx || y >= ny || z >= nz || vals[i] > 2) return ORC_ERR_INVALID_ARG;
        codes[x + (int64_t)nx * (y + (int64_t)ny * z)] = vals[i];
    }
    return ORC_OK;
}

/* ------------------------------------------- map integration */

/* Voxel filter (reading Q33): every point goes to the leaf cell
 * (floor(x/leaf), floor(y/leaf), floor(z/leaf)); each occupied cell yields ONE point,
 * the centroid of its inputs, summed in input order and divided by the count.  Cells
 * are output in ascending (iz, iy, ix) order.  |cell index| must stay below 2^15 - 1 and
 * every coordinate must be finite (INVALID_ARG otherwise).  out_xyz / out_count hold
 * room for n cells; *m_out = number of cells. */
typedef struct { int64_t c[3]; int64_t idx; } orc_cellkey;

static int cellkey_cmp(const void *a, const void *b)
{
    const orc_cellkey *x = (const orc_cellkey *)a, *y = (const orc_cellkey *)b;
    for (int k = 2; k >= 0; --k)
        if (x->c[k] != y->c[k]) return x->c[k] < y->c[k] ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

int orc_voxel_filter(const double *pts, int64_t n, double leaf, double *out_xyz, int32_t *out_count, int64_t *m_out)
{
    if (n < 0 || !(leaf > 0) || !m_out || (n > 0 && (!pts || !out_xyz))) return ORC_ERR_INVALID_ARG;
    *m_out = 0;
    if (n == 0) return ORC_OK;
    orc_cellkey *k = (orc_cellkey *)malloc((size_t)n * sizeof *k);
    if (!k) return ORC_ERR_INVALID_ARG;
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            double v = pts[3 * i + a];
            if (!isfinite(v)) { free(k); return ORC_ERR_INVALID_ARG; }
            double c = floor(v / leaf);
            if (!(fabs(c) < 32767.0)) { free(k); return ORC_ERR_INVALID_ARG; }
            k[i].c[a] = (int64_t)c;
        }
        k[i].idx = i;
    }
    qsort(k, (size_t)n, sizeof *k, cellkey_cmp);
    int64_t m = 0;
    for (int64_t i = 0; i < n;) {
        int64_t j = i;
        double sum[3] = {0.0, 0.0, 0.0};
        while (j < n && k[j].c[0] == k[i].c[0] && k[j].c[1] == k[i].c[1] && k[j].c[2] == k[i].c[2]) {
            for (int a = 0; a < 3; ++a) sum[a] += pts[3 * k[j].idx + a];   /* ascending input index */
            ++j;
        }
        for (int a = 0; a < 3; ++a) out_xyz[3 * m + a] = sum[a] / (double)(j - i);
        if (out_count) out_count[m] = (int32_t)(j - i);
        ++m;
        i = j;
    }
    free(k);
    *m_out = m;
    return ORC_OK;
}

/* World position -> Q16 walk coordinate (reading Q34): round-half-even of
 * ((x - origin) / s) * 65536. */
static int world_to_q16(double x, double origin, double s, int32_t *out)
{
    double q = ((x - origin) / s) * 65536.0;
    if (!(fabs(q) < (double)QLIM)) return ORC_ERR_INVALID_ARG;
    *out = (int32_t)nearbyint(q);
    return ORC_OK;
}

/* Log-odds of a probability, rounded to float (reading Q36). */
static float logodds_f(double p) { return (float)log(p / (1.0 - p)); }

/*
 * Integrate one point cloud into a log-odds store (readings Q33-Q37).
 *
 *   L[x + nx (y + ny z)]  float log-odds per voxel, NaN = never observed (prior P = 0.5)
 *   origin                the sensor position (world)
 *   pts, n                the cloud (world); filtered by orc_voxel_filter when leaf > 0
 *
 * Every (filtered) point p gives the segment origin -> p; if |p - origin| > max_range
 * (> 0) the segment is cut at max_range and carves only (no hit).  Both ends go to Q16
 * (world_to_q16) and the exact DDA of orc_trace_ray lists the voxels the segment
 * visits.  Per cloud every in-grid voxel is updated at most once (Q35): by L_hit if some
 * segment ENDS in it with a hit, else by L_miss if some segment visits it (the end
 * voxel of a cut segment, and the sensor's own voxel, included).  The update is
 * L := clamp((observed ? L : 0) + delta, L_min, L_max) in float.  touched (optional,
 * nx*ny*nz bytes) receives 0 / 1 (miss) / 3 (hit; bit 0 = visited, bit 1 = hit).
 */
int orc_integrate(float *L, int32_t nx, int32_t ny, int32_t nz, double voxel_size, const double map_origin[3],
                  const double origin[3], const double *pts, int64_t n, double p_hit, double p_miss, double p_min,
                  double p_max, double max_range, double leaf, uint8_t *touched, int64_t *n_rays_out)
{
    if (!L || nx < 1 || ny < 1 || nz < 1 || !(voxel_size > 0) || n < 0 || (n > 0 && !pts)) return ORC_ERR_INVALID_ARG;
    if (!(leaf >= 0) || !(p_hit > 0 && p_hit < 1) || !(p_miss > 0 && p_miss < 1) || !(p_min > 0 && p_min < 1) ||
        !(p_max > 0 && p_max < 1) || !(p_min <= p_max))
        return ORC_ERR_INVALID_ARG;
    for (int a = 0; a < 3; ++a)
        if (!isfinite(origin[a])) return ORC_ERR_INVALID_ARG;
    int64_t nvox = (int64_t)nx * ny * nz;
    const double *ray_end = pts;
    double *filt = NULL;
    int64_t m = n;
    if (leaf > 0 && n > 0) {
        filt = (double *)malloc((size_t)n * 3 * sizeof(double));
        int st = orc_voxel_filter(pts, n, leaf, filt, NULL, &m);
        if (st) { free(filt); return st; }
        ray_end = filt;
    } else {
        for (int64_t i = 0; i < 3 * n; ++i)
            if (!isfinite(pts[i])) return ORC_ERR_INVALID_ARG;
    }
    uint8_t *flag = (uint8_t *)calloc((size_t)nvox, 1);
    uint8_t *all_free = (uint8_t *)malloc((size_t)nvox);
    memset(all_free, 1, (size_t)nvox);
    orc_map walk = {nx, ny, nz, voxel_size, {map_origin[0], map_origin[1], map_origin[2]}, {1.0, 1.0, 1.0}, 0,
                    all_free, NULL};
    int status = ORC_OK;
    int32_t o16[3];
    for (int a = 0; a < 3; ++a) status |= world_to_q16(origin[a], map_origin[a], voxel_size, &o16[a]);
    for (int64_t i = 0; i < m && status == ORC_OK; ++i) {
        const double *p = ray_end + 3 * i;
        double d[3] = {p[0] - origin[0], p[1] - origin[1], p[2] - origin[2]};
        double dist = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
        double q[3] = {p[0], p[1], p[2]};
        int hit = 1;
        if (max_range > 0 && dist > max_range) {
            double f = max_range / dist;
            for (int a = 0; a < 3; ++a) q[a] = origin[a] + d[a] * f;
            hit = 0;
        }
        int32_t e16[3];
        for (int a = 0; a < 3; ++a) status |= world_to_q16(q[a], map_origin[a], voxel_size, &e16[a]);
        if (status) break;
        int64_t len = 1;
        for (int a = 0; a < 3; ++a) len += llabs(floor_div(e16[a], QF) - floor_div(o16[a], QF));
        int32_t *ijk = (int32_t *)malloc((size_t)len * 3 * sizeof(int32_t));
        uint8_t *code = (uint8_t *)malloc((size_t)len);
        int32_t got = 0;
        orc_ray r;
        status = orc_trace_ray(&walk, o16, e16, (int32_t)len, ijk, code, &got, &r);
        if (!status && got != len) status = ORC_ERR_SELFCHECK;   /* all-Free map: no early stop */
        for (int64_t s = 0; s < got && !status; ++s) {
            if (code[s] == 255) continue;                           /* outside the grid */
            int64_t v = ijk[3 * s] + (int64_t)nx * (ijk[3 * s + 1] + (int64_t)ny * ijk[3 * s + 2]);
            flag[v] |= (s == got - 1 && hit) ? 3 : 1;
        }
        free(ijk);
        free(code);
    }
    if (status == ORC_OK) {
        float lh = logodds_f(p_hit), lm = logodds_f(p_miss), lo = logodds_f(p_min), hi = logodds_f(p_max);
        for (int64_t v = 0; v < nvox; ++v) {
            if (!flag[v]) continue;
            float l0 = isnan(L[v]) ? 0.0f : L[v];
            float l1 = l0 + ((flag[v] & 2) ? lh : lm);
            if (l1 < lo) l1 = lo;
            if (l1 > hi) l1 = hi;
            L[v] = l1;
        }
        if (touched) memcpy(touched, flag, (size_t)nvox);
    }
    if (n_rays_out) *n_rays_out = m;
    free(flag);
    free(all_free);
    free(filt);
    return status;
}

/* State and probability level of each voxel of a log-odds store (Q37):
 * never observed -> Unknown, level 0; L >= logit(t_occ) -> Occupied; L <= logit(t_free)
 * -> Free; else Unknown; level = number of k in 1..63 with L >= logit((k - 1/2)/63),
 * i.e. round(63 P) with the rounding boundaries taken in log-odds (thresholds rounded
 * to float once). */
void orc_occ_classify(const float *L, int64_t n, double t_occ, double t_free, uint8_t *codes_out,
                      uint8_t *levels_out)
{
    float th_occ = logodds_f(t_occ), th_free = logodds_f(t_free);
    float phi[PLEVELS];
    for (int k = 1; k <= PLEVELS; ++k) phi[k - 1] = logodds_f((k - 0.5) / PLEVELS);
    for (int64_t i = 0; i < n; ++i) {
        float l = L[i];
        if (isnan(l)) {
            codes_out[i] = 0;
            if (levels_out) levels_out[i] = 0;
            continue;
        }
        codes_out[i] = (l >= th_occ) ? 2 : (l <= th_free ? 1 : 0);
        if (levels_out) {
            int lv = 0;
            for (int k = 0; k < PLEVELS; ++k) lv += (l >= phi[k]);
            levels_out[i] = (uint8_t)lv;
        }
    }
}

int orc_version(void) { return 1; }
