/*
 * nbt.h -- C ABI of libnbt, the B200-native online local Information Distribution (ID)
 * of arxiv 2503.22588 ("Next-Best-Trajectory planning ... GPU-parallel online local
 * Information Distribution").  Citations: P:n = /root/reference/PAPER.md line n,
 * S:n = SPEC.md line n, Qn = reading n in DESIGN.md section 2.
 *
 * The library computes, on one CUDA device (sm_100a):
 *   * the voxel-map store (three states, 2-bit packed, L2-resident)
 *   * perspective sampling by Eq. 1
 *   * per-perspective frames and far-plane endpoint lattices
 *   * raycasting with early stop + Eq. 2 scoring
 *   * the per-perspective mean -> the IG point cloud
 *   * the IDW query of Eq. 4 over the last N_B clouds
 *
 * Conventions for every function:
 *   * Return codes only; nothing throws or aborts across the ABI.  On failure a
 *     human-readable detail is available from nbt_last_error_message() (thread-local).
 *   * OWNERSHIP: the library owns everything behind a handle; the caller creates and
 *     destroys handles.  Input arrays are borrowed for the duration of the call only:
 *     host inputs are copied (staged) before the call returns, so the caller may free
 *     or reuse them immediately.  Output arrays are caller-owned.
 *   * "on_device" flags say whether a pointer is device memory of the ctx's device (1)
 *     or host memory (0).  Device pointers must stay valid until the enqueued work
 *     completes.
 *   * ASYNCHRONY: work is enqueued on the ctx stream.  Results written to device
 *     buffers are valid after nbt_ctx_sync() or a sync of that stream.  Results written
 *     to HOST buffers are valid when the call returns (the call synchronizes the
 *     stream).  Calls on one ctx are executed in stream order, so nbt_map_update()
 *     issued after nbt_id_compute() never changes what that compute reads (the
 *     single-writer snapshot rule).
 *   * Validation of host inputs happens before enqueueing and returns the error.
 *     Validation of DEVICE inputs happens on the device: offending elements are
 *     skipped / flagged and the error is returned by the next nbt_ctx_sync().
 *   * A ctx is not thread-safe.  Distinct ctxs share nothing.
 *   * Coordinates: world units (metres in the paper's experiments).  A map maps
 *     world point w to voxel floor((w - origin) / voxel_size) (half-open voxels).
 */
#ifndef NBT_H_
#define NBT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NBT_ABI_VERSION 2

typedef enum {
    NBT_OK = 0,
    NBT_ERR_INVALID_ARG = 1,    /* null pointer, bad size, non-finite value, code >= 3, Q16 overflow */
    NBT_ERR_DEGENERATE = 2,     /* a perspective coincides with the PoI (Q18) */
    NBT_ERR_EMPTY = 3,          /* IDW query on an empty buffer ("no distribution available") */
    NBT_ERR_OUT_OF_MEMORY = 4,
    NBT_ERR_CUDA = 5,           /* a CUDA runtime error; the message names it */
    NBT_ERR_NCCL = 6,           /* reserved for collective failures reported by the caller's layer */
    NBT_ERR_STATE = 7           /* wrong handle state (e.g. map of another ctx) */
} nbt_status;

int         nbt_abi_version(void);
const char *nbt_status_string(nbt_status s);
const char *nbt_last_error_message(void);

/* ---------------------------------------------------------------- context */

typedef struct nbt_ctx_s *nbt_ctx;

/* Bind to CUDA device `device`.  `cuda_stream` is a borrowed cudaStream_t (NULL = the
 * ctx creates and owns a non-blocking stream).  The ctx owns scratch buffers that grow
 * on demand. */
nbt_status nbt_ctx_create(int device, void *cuda_stream, nbt_ctx *out);
/* Replace the borrowed stream (e.g. torch.cuda.current_stream()).  NULL = own stream. */
nbt_status nbt_ctx_set_stream(nbt_ctx ctx, void *cuda_stream);
/* Wait for all enqueued work; returns the first device-side validation error recorded
 * since the previous sync (and clears it), else NBT_OK. */
nbt_status nbt_ctx_sync(nbt_ctx ctx);
void       nbt_ctx_destroy(nbt_ctx ctx);
/* Number of kernels libnbt has launched on this ctx since creation. */
uint64_t   nbt_ctx_launch_count(nbt_ctx ctx);

/* Tuning options of a ctx.  None of them changes any result: every setting gives the
 * same clouds, maps and IDW values bit for bit (the parity tests run the alternatives);
 * they select between measured implementations (knob table).  libnbt
 * reads no environment variable.  NBT_ERR_INVALID_ARG for an unknown option or a value
 * outside its range; get returns the current value. */
enum {
    NBT_OPT_TRACE_REFILL_MIN = 1,   /* idle lanes before a trace warp pops prepared rays: 1..32, default 32 (tile lockstep) */
    NBT_OPT_TRACE_CHUNK_MIN = 2,    /* smallest ray-slot chunk per work grab: 32..1024 (rounded up to 32), default 64 */
    NBT_OPT_TRACE_CARVEOUT = 3,     /* shared-memory carveout (%) of the trace kernel: -1 (driver) .. 100, default 25;
                                       a function attribute, so process-wide: applied at the ctx's next
                                       ID launch (the last ctx to apply a different value sets it) */
    NBT_OPT_DELTA_SORT = 4,         /* 1: map deltas by a CUB radix sort instead of the winner array; default 0 */
    NBT_OPT_FILTER_SORT = 5,        /* 1: the integration's voxel filter by sorting instead of hashing; default 0 */
    NBT_OPT_H2D_MODE = 6,           /* 1: host inputs copied by the driver (pageable) instead of the pinned stage; default 0 */
    NBT_OPT_COPY_THREADS = 7,       /* 0: host staging copies on the caller's thread; 1: chunked over the library's
                                       copy workers (4) while the DMA of landed chunks runs; default 1 on hosts with
                                       >= 8 hardware threads, else 0 */
    NBT_OPT_WALK_WIDTH = 8,         /* decision-term width of nbt_debug_trace: 0 = automatic (int32 unless a
                                       segment has |E_a - O_a| >= 2^30 - 1 Q16 units), 32 or 64 = forced (tests of
                                       the int32 bound; forcing 32 on a longer segment gives NBT_ERR_INVALID_ARG) */
    NBT_OPT_VERBOSE = 9             /* 1: print the trace kernel's occupancy to stderr once; default 0 */
};
nbt_status nbt_ctx_set_option(nbt_ctx ctx, int32_t option, int64_t value);
nbt_status nbt_ctx_get_option(nbt_ctx ctx, int32_t option, int64_t *value);

/* Optional per-kernel device timing with CUDA events recorded on the ctx stream around
 * each launch of the named kernel family (used by bench.py for the roofline). */
enum {
    NBT_KERNEL_TRACE = 0,       /* k_id_trace: rows a5-a8, the hot loop */
    NBT_KERNEL_FRAMES = 1,      /* k_persp_frames: row a4 */
    NBT_KERNEL_FINALIZE = 2,    /* k_id_finalize: row a8 */
    NBT_KERNEL_IDW = 3,         /* k_idw_query: row a9 */
    NBT_KERNEL_SAMPLE = 4,      /* k_sample_perspectives: row a3 */
    NBT_KERNEL_MAP_UPDATE = 5,  /* k_delta_win + k_delta_apply_win (or the sort form): row a2 */
    NBT_KERNEL_INTEGRATE = 6,   /* voxel filter + k_integrate_rays + k_integrate_apply: row f3 */
    NBT_KERNEL_COUNT = 7
};
nbt_status nbt_ctx_set_profiling(nbt_ctx ctx, int enable);
/* Record only the kernel families whose bit (1 << NBT_KERNEL_*) is set (0 = off).  Inside a
 * graph every recorded family adds two event nodes (~2 us each on B200), so a timed graph
 * should record no more than the families it reports. */
nbt_status nbt_ctx_set_profiling_mask(nbt_ctx ctx, uint32_t kernel_mask);
/* Sum of the recorded durations (ms) and number of launches of `kernel` since the last
 * reset; synchronizes the stream.  reset != 0 clears the record. */
nbt_status nbt_ctx_profile_read(nbt_ctx ctx, int32_t kernel, double *total_ms, uint64_t *launches, int reset);

/* CUDA-graph capture of a sequence of calls on the ctx (an MHP cycle with device-resident
 * inputs and outputs), replayed with one launch.  Between begin and end, calls are
 * RECORDED, not executed: only device pointers are allowed (host inputs or outputs give
 * NBT_ERR_STATE), and scratch buffers must already have their size (run the sequence
 * once before capturing).  The ID ring buffer keeps its state on the device, so replays
 * push and query correctly.  Kernel parameters (PoI, seeds, pointers) are fixed at
 * capture time.  With profiling on, the captured kernels are bracketed by event nodes
 * whose times nbt_graph_profile_read returns for the last replay. */
typedef struct nbt_graph_s *nbt_graph;
nbt_status nbt_ctx_capture_begin(nbt_ctx ctx);
nbt_status nbt_ctx_capture_end(nbt_ctx ctx, nbt_graph *out);
nbt_status nbt_graph_launch(nbt_graph graph);
/* Sum of the last replay's durations (ms) of the captured launches of `kernel`; syncs. */
nbt_status nbt_graph_profile_read(nbt_graph graph, int32_t kernel, double *total_ms, uint64_t *launches);
void       nbt_graph_destroy(nbt_graph graph);

/* ------------------------------------------------------- voxel map (row a1, a2) */

enum { NBT_UNKNOWN = 0, NBT_FREE = 1, NBT_OCCUPIED = 2 };      /* three states (Eq. 2) */
enum { NBT_OUTSIDE_UNKNOWN = 0, NBT_OUTSIDE_CLIP = 1 };        /* Q14 */
/* Store layouts: linear x-fastest inside a sentinel shell (default), or a
 * Morton cube (bit-interleaved coordinates; a 128-B line is an 8x8x8 block). */
enum { NBT_LAYOUT_LINEAR = 0, NBT_LAYOUT_MORTON = 1 };

typedef struct nbt_map_s *nbt_map;

typedef struct {
    int32_t nx, ny, nz;       /* voxels per axis, each >= 1; (nx+32)(ny+32)(nz+32) < 2^32
                                 (< 2^31 for the 2-bit linear store) */
    double  voxel_size;       /* s_Vox > 0 (1 cm) */
    double  origin[3];        /* world position of voxel (0,0,0)'s min corner */
    double  gain[3];          /* g[U], g[F], g[O] of Eq. 2 as per-state constants (Q15);
                                 default {1.0, 0.12, 0.03}; each finite, >= 0 */
    int32_t outside_policy;   /* NBT_OUTSIDE_UNKNOWN (default) or NBT_OUTSIDE_CLIP */
    int32_t layout;           /* NBT_LAYOUT_LINEAR (default) or NBT_LAYOUT_MORTON (the Morton cube must
                                 fit 1024^3 voxels and 8x the linear store, else NBT_ERR_INVALID_ARG) */
    int32_t state_bits;       /* bits per voxel of nbt_map_create: 2 (default: 16 voxels per 32-bit
                                 word) or 8 (one byte per voxel); nbt_map_create_prob always uses 8 */
} nbt_map_desc;

/* Fill *desc with the defaults above for an nx*ny*nz grid of voxel_size at origin 0. */
void nbt_map_desc_default(nbt_map_desc *desc, int32_t nx, int32_t ny, int32_t nz, double voxel_size);
/* Create a map whose every voxel is Unknown (UFOMap's default). */
nbt_status nbt_map_create(nbt_ctx ctx, const nbt_map_desc *desc, nbt_map *out);
/* Create a map that also stores each voxel's occupancy probability, so the ID scores every
 * voxel by Eq. 2 exactly: Unknown 1, Free P, Occupied 1 - P,
 * with P quantised to k/63 (reading Q32) and desc->gain unused by the ID.  8 bits per voxel.
 * State-only writes (nbt_map_upload, nbt_map_update) store P_F = gain[1], P_O = 1 - gain[2]. */
nbt_status nbt_map_create_prob(nbt_ctx ctx, const nbt_map_desc *desc, nbt_map *out);
/* Replace all voxels: codes[x + nx*(y + ny*z)] in {0,1,2}; n must equal nx*ny*nz.
 * Synchronizes the ctx stream; a code >= 3 gives NBT_ERR_INVALID_ARG (map unchanged
 * for host input; for device input the offending voxels become Unknown). */
nbt_status nbt_map_upload(nbt_map map, const uint8_t *codes, size_t n, int on_device);
/* Replace all voxels from occupancy probabilities (Q16): observed[i] == 0 ->
 * Unknown; p[i] >= t_occ -> Occupied; p[i] <= t_free -> Free; else Unknown. */
nbt_status nbt_map_upload_prob(nbt_map map, const float *p, const uint8_t *observed, size_t n,
                               int on_device, double t_occ, double t_free);
/* Per-voxel-probability deltas (maps of nbt_map_create_prob; on a state-only map the
 * probabilities are ignored): voxel i := classify(p[i], observed[i]) by S:69 with the
 * probability level round-half-even(63 clamp(p, 0, 1)).  Same ordering and validation as
 * nbt_map_update. */
nbt_status nbt_map_update_prob(nbt_map map, const int32_t *ijk, const float *p, const uint8_t *observed, size_t n,
                               int on_device, double t_occ, double t_free);
/* Apply n sparse deltas: voxel (ijk[3i], ijk[3i+1], ijk[3i+2]) := codes[i].  Indices must
 * lie inside the grid and codes in {0,1,2}.  Duplicated voxels resolve to the LAST delta
 * in array order (Q30).  Stream-ordered after earlier work on the ctx.  n == 0 is a no-op. */
nbt_status nbt_map_update(nbt_map map, const int32_t *ijk, const uint8_t *codes, size_t n, int on_device);
/* Device pointer and size of the packed store (for an in-place NCCL broadcast of a
 * replica; every replica has the same layout for the same desc). */
nbt_status nbt_map_device_buffer(nbt_map map, void **dev_ptr, size_t *bytes);
/* Unpack to dense x-fastest uint8 codes (host buffer of n = nx*ny*nz bytes); syncs. */
nbt_status nbt_map_download(nbt_map map, uint8_t *codes_out, size_t n);
/* Probability levels (P = level / 63; 0 for Unknown) of a nbt_map_create_prob map; syncs. */
nbt_status nbt_map_download_levels(nbt_map map, uint8_t *levels_out, size_t n);
/* Copy of the descriptor. */
nbt_status nbt_map_get_desc(nbt_map map, nbt_map_desc *out);
void       nbt_map_destroy(nbt_map map);

/* ------------------------------------------- map integration */

/* The step before the ID: a depth frame is thinned by a voxel filter
 * and integrated into a probabilistic occupancy store by log-odds hit / miss updates with
 * free-space carving along the sensor rays (the paper defers the occupancy
 * model to its mapping framework).  The store keeps float32 log-odds per voxel
 * (NaN = never observed, reading Q36); every integration also writes the resulting
 * state (and, for a nbt_map_create_prob map, the probability level) of each changed
 * voxel into an ID map on the device and records those changes as a2 deltas. */
typedef struct nbt_occ_s *nbt_occ;

typedef struct {
    double p_hit, p_miss;     /* hit / miss probabilities: 0.7, 0.4 */
    double p_min, p_max;      /* clamp: 0.12, 0.97 */
    double t_occ, t_free;     /* state thresholds: 0.5, 0.5 */
    double max_range;         /* r_max, world units; a farther point is cut there and only
                                 carves; <= 0 = unlimited; default 5.0 */
    double leaf;              /* voxel-filter leaf, world units; 0 = no filter (Q33);
                                 default = the map's voxel size */
} nbt_integrate_params;

/* Fill *p with the defaults above for a map of the given voxel size. */
void nbt_integrate_params_default(nbt_integrate_params *p, double voxel_size);

/* Occupancy store over desc's grid (nx*ny*nz < 2^31), every voxel never observed.
 * Owns ~15 bytes of device memory per voxel (log-odds, flag byte, voxel and delta lists). */
nbt_status nbt_occ_create(nbt_ctx ctx, const nbt_map_desc *desc, nbt_occ *out);
/* Replace / read all log-odds (dense x-fastest float32, NaN = never observed); n must be
 * nx*ny*nz.  Upload is stream-ordered (host input is staged); download syncs. */
nbt_status nbt_occ_upload(nbt_occ occ, const float *logodds, size_t n, int on_device);
nbt_status nbt_occ_download(nbt_occ occ, float *logodds_out, size_t n);
/* Integrate one cloud of n points (xyz float64, world units; host or device memory)
 * seen from sensor[3] (host).  prm NULL = defaults.  Each (filtered) point gives the ray
 * sensor -> point walked by the exact DDA of the ID (Q34); per call each in-grid voxel
 * is updated once: by the hit if some ray ends in it, else by the miss if some ray
 * visits it (Q35); L := clamp(L + delta) in float (Q36).  map (NULL allowed; same nx,
 * ny, nz) receives the new state -- L >= logit(t_occ) Occupied, <= logit(t_free) Free,
 * else Unknown -- and level round(63 P) (Q37) of every voxel whose (state, level)
 * changed.  A non-finite point, a leaf cell index |c| >= 2^15 - 1 or a Q16 overflow makes the
 * whole call a no-op, reported as NBT_ERR_INVALID_ARG by the next nbt_ctx_sync or
 * nbt_occ_stats (points are validated on the device).  n < 2^31.  Stream-ordered; host
 * points are staged through pinned memory, no sync. */
nbt_status nbt_occ_integrate(nbt_occ occ, nbt_map map, const double sensor[3], const double *points, int64_t n,
                             int on_device, const nbt_integrate_params *prm);
/* Counters of the last integrate (syncs): out[0] input points, out[1] rays after the
 * filter, out[2] voxels updated, out[3] a2 deltas emitted. */
nbt_status nbt_occ_stats(nbt_occ occ, int64_t out[4]);
/* The a2 deltas of the last integrate, in unspecified order (syncs): voxel (ijk[3i],
 * ijk[3i+1], ijk[3i+2]) now has state codes[i] and level levels[i] (0 if never
 * observed).  Copies min(cap, count) entries; *n_out = count. */
nbt_status nbt_occ_deltas(nbt_occ occ, int32_t *ijk, uint8_t *codes, uint8_t *levels, size_t cap, size_t *n_out);
void       nbt_occ_destroy(nbt_occ occ);

/* The voxel filter alone (Q33): one centroid per occupied leaf cell, cells in
 * ascending (iz, iy, ix) order; out_xyz (3 n doubles) and out_count (n, may be NULL) are
 * host buffers; *m_out = number of cells.  Syncs. */
nbt_status nbt_voxel_filter(nbt_ctx ctx, const double *points, int64_t n, int on_device, double leaf,
                            double *out_xyz, int32_t *out_count, int64_t *m_out);

/* ------------------------------------------------------------ camera (row a5) */

typedef struct {
    int32_t width, height;          /* ray lattice W x H (>= 1 each) */
    double  fx, fy, cx, cy;         /* pinhole intrinsics, pixel units; 2cx = W-1, 2cy = H-1 */
    int32_t add_corners;            /* 1 = append the 4 far-plane corner rays (s_G mode) */
    double  tan_half_fov_h, tan_half_fov_v;   /* tan(FoV/2), used for the corner rays */
} nbt_camera;

/* Corner-inclusive W x H lattice spanning the FoV on the far plane at d_Cam:
 * ray (i, kk) ends at  p_P + d_Cam*fwd + (i-cx)/fx*d_Cam*right + (kk-cy)/fy*d_Cam*up,
 * fx = (W-1)/(2 tan(FoV_h/2)) (1 if W = 1), so pixels 0 and W-1 lie on d_h. */
nbt_status nbt_camera_from_fov(double fov_h, double fov_v, int32_t w, int32_t h, nbt_camera *out);
/* The paper's s_G lattice: spacing s_G*voxel_size on the far plane, centred,
 * plus the 4 corner rays unless they coincide with lattice points (Q6-Q9). */
nbt_status nbt_camera_from_grid_scaling(double fov_h, double fov_v, double range, double voxel_size,
                                        double s_g, nbt_camera *out);
/* N_E = W*H (+4 with corners). */
int32_t    nbt_camera_num_rays(const nbt_camera *cam);

/* ------------------------------------------------------ perspectives (row a3) */

enum { NBT_SAMPLE_BALL = 0, NBT_SAMPLE_SURFACE = 1 };
/* Eq. 1 (Q1-Q3, Q29): n points p = poi + r_s * X_R^(1/3) * X/|X| written to
 * xyz_out (n x 3 doubles, row-major), on the device (out_on_device = 1) or the host. */
nbt_status nbt_sample_perspectives(nbt_ctx ctx, const double poi[3], double r_s, int32_t n, uint64_t seed,
                                   int32_t mode, double *xyz_out, int out_on_device);

/* ----------------------------------------- the Information Distribution (a4-a8) */

typedef struct {
    double   *xyz;        /* n x 3: the perspective origins p_P,j (copied from the input) */
    double   *gain;       /* n: g_P,j, canonical form Q26 */
    uint64_t *counts;     /* n x 4 or NULL: T_U, T_F, T_O (per-state visit totals over the
                             perspective's rays) and L (in-grid lookups) */
    int32_t   on_device;  /* 1: the three buffers are device memory of the ctx's device */
} nbt_ig_cloud;

/* The ID: for each perspective j of persp_xyz (n_persp x 3), cast the
 * camera's N_E rays of length `range` (d_Cam, world units) towards the PoI through the
 * map, stop each at its first Occupied voxel, score visited voxels by Eq. 2 and average
 * per perspective.  Output row j belongs to input row j.  Errors: NBT_ERR_DEGENERATE if
 * a host perspective equals the PoI (Q18); NBT_ERR_INVALID_ARG for non-finite inputs or
 * a Q16 coordinate outside (-2^30, 2^30) (Q19).  n_persp == 0 is a no-op. */
nbt_status nbt_id_compute(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                          int32_t n_persp, int persp_on_device, const nbt_camera *cam, double range,
                          nbt_ig_cloud *out);
/* Shard form for multi-GPU: computes only perspectives j = first + i*stride
 * (i = 0, 1, ...) and writes them COMPACTLY to out rows i. */
nbt_status nbt_id_compute_slice(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                                int32_t n_persp, int persp_on_device, int32_t first, int32_t stride,
                                const nbt_camera *cam, double range, nbt_ig_cloud *out);

/* Ray-split form for multi-GPU when perspectives are fewer than GPUs (SURVEY 8e "ray-split
 * fallback"): the rays of EVERY perspective are dealt to ray_world shards and this call
 * walks shard ray_rank's rays only.  Units of 32 rays: with W >= 8 and H >= 4 the 8x4
 * pixel tiles (tx, ty) = (i / 8, kk / 4), unit u = ty * ceil(W / 8) + tx; otherwise
 * u = floor(k / 32) for the row-major ray index k = kk * W + i (Q27).  Shard r walks the
 * units u with u mod ray_world == r; the 4 corner rays of the s_G mode belong to shard 0.
 * totals_out: DEVICE memory of the ctx's device, n_persp x NBT_ID_TOTALS uint64 per
 * perspective = (T_U, T_F, T_O, L, T_G) over this shard's rays (T_G: the Eq. 2 gain in 1/63
 * units, Q32; meaningful only for a per-voxel-probability map, ignore it otherwise),
 * overwritten.  The totals are
 * integers, so their sum over the shards (e.g. an all-reduce) equals the whole ID's totals
 * exactly; nbt_id_finalize turns them into the IG cloud.  Validation as nbt_id_compute;
 * NBT_ERR_INVALID_ARG unless 0 <= ray_rank < ray_world and totals_out is device memory. */
#define NBT_ID_TOTALS 5
nbt_status nbt_id_compute_rays(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                               int32_t n_persp, int persp_on_device, int32_t ray_rank, int32_t ray_world,
                               const nbt_camera *cam, double range, uint64_t *totals_out);
/* The IG cloud of the totals summed over all ray shards (Q26/Q32), the same fp64
 * expression nbt_id_compute ends with, so the result is bit-identical to nbt_id_compute on
 * one GPU.  totals: DEVICE memory, n_persp x NBT_ID_TOTALS uint64 (read only); the
 * perspectives are validated again (a degenerate one gets NBT_ERR_DEGENERATE / NaN, as in
 * nbt_id_compute). */
nbt_status nbt_id_finalize(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                           int32_t n_persp, int persp_on_device, const nbt_camera *cam, double range,
                           const uint64_t *totals, nbt_ig_cloud *out);

/* Peer-memory gather of the IG cloud (one process per GPU): the all-gather after
 * the sharded ID is fused into the finalize kernel, which stores every computed row straight
 * into each rank's row buffer (other GPUs' buffers mapped with CUDA IPC, so the stores cross
 * NVLink/NVSwitch; on one GPU shared by several processes they are plain device stores).
 *   nbt_gather_create   this rank's buffer for the whole cloud: `rows` rows, owned by the
 *                       handle (device memory, one cudaMalloc); world <= 16, 0 <= rank < world.
 *   nbt_gather_export   its CUDA IPC handle (NBT_PEER_HANDLE_BYTES opaque bytes) for the peers.
 *   nbt_gather_attach   map peer_rank's exported buffer (a handle from ANOTHER process; this
 *                       rank's own entry needs no attach).  NBT_ERR_CUDA if IPC is unavailable.
 *   nbt_gather_rows     device pointers of this rank's buffer as a cloud (xyz rows x 3, gain
 *                       rows, counts rows x 4; on_device = 1), e.g. for nbt_idbuf_push.
 *   nbt_id_compute_gather  nbt_id_compute_slice(first, stride) whose finalize writes the row
 *                       of perspective j = first + i*stride (of persp_xyz, n_persp rows) to row
 *                       row0 + j of EVERY rank's buffer: row0 = 0 with the whole perspective
 *                       set on every rank (strided shards), row0 = rank * n with each rank's
 *                       own n perspectives (weak scaling).  NBT_ERR_INVALID_ARG unless
 *                       row0 + n_persp <= rows; every rank must be attached (NBT_ERR_STATE).
 * Ordering is the caller's: a rank may read its buffer after every rank's call has completed
 * (e.g. each rank synchronises its stream, then a process barrier), and a buffer must not be
 * rewritten while a peer may still read it (alternate two gathers between cycles). */
#define NBT_PEER_HANDLE_BYTES 64
typedef struct nbt_gather_s *nbt_gather;
nbt_status nbt_gather_create(nbt_ctx ctx, int32_t rows, int32_t world, int32_t rank, nbt_gather *out);
nbt_status nbt_gather_export(nbt_gather g, uint8_t handle_out[NBT_PEER_HANDLE_BYTES]);
nbt_status nbt_gather_attach(nbt_gather g, int32_t peer_rank, const uint8_t handle[NBT_PEER_HANDLE_BYTES]);
nbt_status nbt_gather_rows(nbt_gather g, nbt_ig_cloud *rows_out);
nbt_status nbt_id_compute_gather(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                                 int32_t n_persp, int persp_on_device, int32_t first, int32_t stride,
                                 int32_t row0, const nbt_camera *cam, double range, nbt_gather g);
/* Ray split with the all-reduce fused into the walk (N_P < G): like
 * nbt_id_compute_rays with ray_rank = the gather's rank and ray_world = its world, but the
 * walk's count flushes add straight into EVERY rank's buffer, read as n_persp x NBT_ID_TOTALS
 * uint64 totals at its start (remote atomics over the peer mappings; n_persp * 40 bytes must
 * fit rows * 64).  Each rank first clears its own buffer with nbt_gather_zero; the caller
 * orders all ranks' clears before any rank's call and all calls before the readers (e.g. a
 * stream-ordered all-reduce of one word), then nbt_id_finalize turns a buffer's summed totals
 * into the cloud -- bit-identical to nbt_id_compute on one GPU. */
nbt_status nbt_gather_zero(nbt_gather g);
nbt_status nbt_id_compute_rays_gather(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                                      int32_t n_persp, int persp_on_device, const nbt_camera *cam, double range,
                                      nbt_gather g);
void       nbt_gather_destroy(nbt_gather g);

/* -------------------------------------------- ID buffer + IDW query (row a9) */

typedef struct nbt_idbuf_s *nbt_idbuf;

/* Device ring buffer of the last `capacity_nb` IG clouds (N_B = 10 in P:310), each of
 * at most max_persp perspectives. */
nbt_status nbt_idbuf_create(nbt_ctx ctx, int32_t capacity_nb, int32_t max_persp, nbt_idbuf *out);
/* Copy a cloud (n perspectives: xyz + gain) in as the NEWEST entry; evicts the oldest
 * when full.  Stream-ordered. */
nbt_status nbt_idbuf_push(nbt_idbuf buf, const nbt_ig_cloud *cloud, int32_t n);
nbt_status nbt_idbuf_clear(nbt_idbuf buf);
int32_t    nbt_idbuf_size(nbt_idbuf buf);
/* Eq. 4 at n_q query positions (n_q x 3): G(x) = sum_u w_u v_u(x), entries u =
 * oldest..newest, w_u = 1/(m-u) (newest 1, Q21), v_u = sum_j g_j d_j^-p / sum_j d_j^-p
 * over entry u's perspectives (Q20, Q22), v_u = gain of the nearest perspective if its
 * distance < zero_eps (Q23).  normalize_weights != 0 divides by sum_u w_u.  g_out has n_q
 * doubles on the device (out_on_device = 1) or the host.  NBT_ERR_EMPTY if no entry. */
nbt_status nbt_ig_query(nbt_idbuf buf, const double *query_xyz, int32_t n_q, int q_on_device,
                        double power_p, double zero_eps, int32_t normalize_weights,
                        double *g_out, int out_on_device);
/* Eq. 4 over the knn nearest perspectives of each entry only (reading Q22, the optional
 * "nearest perspectives" form of P:274): nearest by squared distance, ties to the lower
 * index; knn in [1, 16]; knn = 0 is nbt_ig_query.  Same arguments and errors otherwise. */
nbt_status nbt_ig_query_knn(nbt_idbuf buf, const double *query_xyz, int32_t n_q, int q_on_device,
                            double power_p, double zero_eps, int32_t normalize_weights, int32_t knn,
                            double *g_out, int out_on_device);
void       nbt_idbuf_destroy(nbt_idbuf buf);

/* The MHP's information cost over candidate trajectories:
 * for n_traj trajectories of poses_per_traj camera poses each (K + 1 = 31 in P:309),
 * pose i = (pose_xyz[3i..], pose_axis[3i..] = optical axis, any length > 0):
 *   O_i = cos(theta_i) if theta_i <= theta_cut else 0, theta_i = angle(axis_i, PoI - pos_i)
 *         (the FoV cut as cos(theta_i) >= cos_theta_cut, reading Q31),
 *   G_i = the IDW value of nbt_ig_query at pos_i,
 *   c_out[t] = sum over the trajectory's poses, in order, of w_i / (O_i * G_i + eps)
 *         (eps = 1e-7 in P:259).
 * o_out / g_out (n_traj * poses_per_traj doubles) may be NULL.  NBT_ERR_DEGENERATE if a
 * host pose lies within 1e-9 of the PoI (device poses: flagged, reported by the next
 * nbt_ctx_sync and their outputs are NaN).  NBT_ERR_EMPTY on an empty buffer. */
nbt_status nbt_info_cost(nbt_idbuf buf, const double *pose_xyz, const double *pose_axis, int32_t n_traj,
                         int32_t poses_per_traj, int poses_on_device, const double poi[3], double cos_theta_cut,
                         double w_i, double eps, double power_p, double zero_eps, int32_t normalize_weights,
                         double *o_out, double *g_out, double *c_out, int out_on_device);

/* ----------------------------------------------------------- test hooks */

/* Per-ray walk of explicit segments in Q16 voxel coordinates (65536 units per voxel,
 * reading Q19; host arrays, n_rays x 3 int32 each, inside (-2^30, 2^30)): the first
 * max_visits visited voxels of ray r go to ijk_out[r*max_visits*3 ...], their codes
 * (0/1/2; 255 = outside the grid) to code_out[r*max_visits ...]; len_out[r] = number of
 * visited voxels (may exceed max_visits); counts_out[r*4 ...] = n_U, n_F, n_O, lookups.
 * Uses the same device traversal as nbt_id_compute.  Synchronizes. */
nbt_status nbt_debug_trace(nbt_ctx ctx, nbt_map map, const int32_t *o_q16, const int32_t *e_q16,
                           int32_t n_rays, int32_t max_visits, int32_t *ijk_out, uint8_t *code_out,
                           int32_t *len_out, uint32_t *counts_out);
/* Per-ray counts of the PRODUCTION trace (the k_id_trace code nbt_id_compute runs, in an
 * instance that also records every closed ray): n host perspectives, the same arguments as
 * nbt_id_compute; ray_counts_out (host, n x N_E x 5 uint32) receives for ray k of perspective
 * j (Q27 order: row-major lattice rows, then the 4 corner rays) its n_U, n_F, n_O, in-grid
 * lookups and stop flag (1 = stopped on an Occupied voxel).  Synchronizes. */
nbt_status nbt_debug_id_rays(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz, int32_t n,
                             const nbt_camera *cam, double range, uint32_t *ray_counts_out);
/* The device frames of n perspectives (host in/out): 18 int32 per perspective
 * (O, A, Rh, Uh, Rc, Uc, each xyz) and a status per perspective (0 ok). Synchronizes. */
nbt_status nbt_debug_frames(nbt_ctx ctx, nbt_map map, const double poi[3], const double *persp_xyz,
                            int32_t n, const nbt_camera *cam, double range, int32_t *q16_out,
                            int32_t *status_out);

#ifdef __cplusplus
}
#endif
#endif /* NBT_H_ */
