/*
 * cil.h -- C ABI of the B200-native ICP hot path (libcil.so).
 *
 * The operation is one rigid ICP iteration as the cilantro paper (arXiv 1807.00399)
 * states it: "the top-level loop logic (alternating between correspondence estimation
 * and transformation parameter optimization) of the Iterative Closest Point (ICP)
 * algorithm ... parameterized by the correspondence estimation mechanism and the transform
 * estimator ... a standard, kd-tree based correspondence search engine ... optimizers for
 * rigid [Besl & McKay; Low] ... registration under the point-to-point and point-to-plane
 * metrics" (section "Functionality / Iterative geometric registration"),
 * run with "nearest neighbor kd-tree queries, with a rejection distance threshold" and
 * "a fixed number of ... iterations" (section "Performance").
 * Inputs are matrix views with "one data point per column ... contiguously stored in
 * memory, in column-major order": for D = 3 this is packed fp32 x,y,z,x,y,z...
 *
 * Conventions (every function):
 *   - Every array pointer is a DEVICE pointer unless stated otherwise.  Calls are
 *     stream-ordered and asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) and never synchronise the device.
 *   - Points and normals: packed fp32 xyz, element i at [3*i .. 3*i+2], 4-byte aligned.
 *   - Poses: 4x4 row-major fp64 matrices mapping SOURCE coordinates to TARGET coordinates,
 *     [R t; 0 0 0 1] (reading R5: increments are left-composed).
 *   - Counts n, m: 0 <= m, 1 <= n, both <= INT32_MAX.
 *   - Ownership: the caller owns every input, output and workspace buffer; the library
 *     keeps no caller pointer beyond the enqueued work.  A cil_target owns its device
 *     buffers (allocated stream-ordered on the build stream, freed by cil_target_free).
 *     A built target is immutable: concurrent queries on different streams are allowed,
 *     each with its own workspace; a workspace must not be shared by concurrent calls.
 *   - Errors: host-detectable problems (NULL pointers, bad sizes or parameters, missing
 *     normals for point-to-plane, small or misaligned workspace, CUDA launch failures)
 *     are returned synchronously, before anything is enqueued when possible.  Data-
 *     dependent outcomes (degenerate 6x6 system, zero correspondences) are written on the
 *     device into the .status field of the result/system structs.  The library never
 *     aborts and never prints.  cil_last_error() gives a thread-local detail string.
 *   - No CPU fallback exists: every step runs in the library's own sm_100a kernels.
 */
#ifndef CIL_H_
#define CIL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A cudaStream_t (identical type: pointer to the opaque CUDA stream struct). */
typedef struct CUstream_st* cil_stream_t;

typedef enum {
    CIL_OK = 0,
    CIL_ERR_INVALID_ARG = 1,   /* NULL pointer, n/m out of range, bad metric, max_dist <= 0 ... */
    CIL_ERR_EMPTY_TARGET = 2,  /* n == 0 ("errors: empty target") */
    CIL_ERR_NO_NORMALS = 3,    /* point-to-plane on a target built without normals */
    CIL_ERR_CUDA = 4,          /* a CUDA runtime call or launch failed; see cil_last_error() */
    CIL_ERR_OOM = 5,           /* device allocation failed */
    CIL_ERR_WORKSPACE = 6,     /* ws NULL, misaligned (needs 256 B) or smaller than required */
    /* reported on the device in cil_icp_result.status / cil_icp_system.status: */
    CIL_ERR_DEGENERATE = 16,       /* count < 6, Cholesky pivot <= 0 or min/max pivot < 1e-12 (R9) */
    CIL_NO_CORRESPONDENCES = 17    /* no pair within max_corr_dist (R10) */
} cil_status;

typedef enum {
    CIL_POINT_TO_POINT = 0,    /* r = s - t,        J = [-[s]x , I3]  [Besl & McKay]  */
    CIL_POINT_TO_PLANE = 1,    /* r = (s - t).n,    J = [s x n ; n]   [Low 2004]      */
    CIL_COMBINED = 2           /* w_point |s - t|^2 + w_plane ((s - t).n)^2: the weighted
                                  combination the paper names (R22) */
} cil_metric;

typedef struct cil_target cil_target;   /* opaque, immutable after build */

/* Spatial index kinds (BASELINE.json north_star (2): "a uniform grid or Morton-sorted cells
   ... or a GPU-traversable kd-tree, chosen by measurement"; DESIGN.md 4.1b has the table). */
typedef enum {
    CIL_INDEX_BVH = 0,     /* Morton-sorted leaves + implicit binary BVH (default; every path) */
    CIL_INDEX_GRID = 1     /* the BVH plus a uniform grid (cells sized for grid_points targets per
                              cell from the bounding box; capped at 2n cells): cil_nn_query and the
                              stateless cil_icp_iterate search the grid (shells of cells, exact;
                              lanes still unresolved after 2 shells finish on the BVH); the
                              certified loop (cil_icp_run, shards) keeps the BVH.  Fastest when the
                              target fills its bounding box and queries lie inside it (C2) */
} cil_index_kind;

/* Spatial-index parameters (NULL = defaults).  leaf_size: points per BVH leaf
   (0 = default 16; 4, 8, 16 or 32).  index_kind: cil_index_kind.  grid_points: mean target
   points per grid cell over the bounding box (0 = default 1; CIL_INDEX_GRID only; > 0 and
   finite).  Other fields reserved, must be 0. */
typedef struct {
    int32_t leaf_size;
    int32_t index_kind;
    float grid_points;
    int32_t reserved[5];
} cil_index_params;

/* ICP parameters.  metric: cil_metric.  max_iters >= 1 (cil_icp_run only).
   max_corr_dist > 0: pairs with |s - t| > max_corr_dist are rejected (inclusive bound,
   PAPER.md:195, R2).  rot_tol (rad) / trans_tol: cil_icp_run stops after an
   iteration whose increment has angle < rot_tol AND |tau| < trans_tol (both 0 = fixed
   iteration count).  w_point/w_plane: the weights of CIL_COMBINED (finite,
   >= 0, not both 0; H = w_point H_point + w_plane H_plane, likewise g and the squared-residual
   sum); must be 0 for the single metrics.  Point-to-plane and combined need target normals. */
typedef struct {
    int32_t metric;
    int32_t max_iters;
    double max_corr_dist;
    double rot_tol;
    double trans_tol;
    double w_point;
    double w_plane;
} cil_icp_params;

/* Result of cil_icp_run, written on the device.  rmse = sqrt(sum r^2 / n_corr) over the
   accepted pairs of the last executed iteration, before its update (R11); iterations =
   number of executed iterations (an iteration that finds no pair or a degenerate system
   counts, and stops the loop with the pose unchanged). */
typedef struct {
    double pose[16];
    double rmse;
    int64_t n_corr;
    int32_t iterations;
    int32_t converged;
    int32_t status;     /* CIL_OK, CIL_ERR_DEGENERATE or CIL_NO_CORRESPONDENCES */
    int32_t pad;
} cil_icp_result;

/* The normal equations of one iteration, written on the device: H (6x6 row-major,
   symmetric), g (6), sse = sum of squared residuals, n_corr accepted pairs; x = the
   increment -H^-1 g (alpha = x[0:3], tau = x[3:6]; zeros when status != CIL_OK). */
typedef struct {
    double H[36];
    double g[6];
    double x[6];
    double sse;
    int64_t n_corr;
    int32_t status;
    int32_t pad;
} cil_icp_system;

/* Host-readable description of a built target. */
typedef struct {
    int64_t n;            /* number of target points */
    int64_t n_leaves;     /* BVH leaves */
    int64_t n_nodes;      /* implicit binary-tree node slots (2 * next_pow2(n_leaves)) */
    int32_t leaf_size;
    int32_t has_normals;
    int64_t device_bytes; /* bytes owned by the target */
    int32_t index_kind;   /* cil_index_kind it was built with */
    int32_t pad;
} cil_target_info;

/* Build the spatial index over the target (BASELINE.json north_star
   "(2) a GPU spatial index over the target ... Morton-sorted cells built by a device radix
   sort"): bounding box -> 63-bit Morton keys -> radix sort -> reorder points/normals ->
   leaf and node AABBs of an implicit binary BVH.
   pts [n*3] fp32 device; normals [n*3] fp32 device or NULL (required for point-to-plane).
   On success *out receives the new target (host handle).  The inputs may be freed after
   the stream reaches the end of the enqueued work. */
cil_status cil_target_build(const float* pts, const float* normals, int64_t n,
                            const cil_index_params* params, cil_stream_t stream, cil_target** out);

/* Release a target (stream-ordered free on `stream`). NULL is a no-op. */
cil_status cil_target_free(cil_target* t, cil_stream_t stream);

/* Host-only: describe a target. */
cil_status cil_target_get_info(const cil_target* t, cil_target_info* info);

/* Exact 1-NN ("k-NN ... queries"): for each query q_i
   (packed fp32 xyz [m*3]) find argmin_j |q_i - t_j|^2 over the target, ties to the lowest
   ORIGINAL target index (R1).  max_dist: only targets with |q - t| <= max_dist count
   (INFINITY = unbounded).  Outputs in query order: idx[m] int32 original target index or -1,
   sqdist[m] fp32 squared distance or +INF (BASELINE.json configs[1] "output nearest index
   (int32) and squared distance").  Either output may be NULL. m == 0 is a no-op. */
cil_status cil_nn_query(const cil_target* t, const float* queries, int64_t m, float max_dist,
                        int32_t* idx, float* sqdist, cil_stream_t stream);

/* Host-only: exact workspace size in bytes for cil_icp_iterate / cil_icp_run on m
   source points (the same size serves both).  Returns 0 for invalid arguments. */
size_t cil_icp_workspace_bytes(int64_t m, const cil_icp_params* params);

/* One stateless ICP iteration: s_i = R p_i + t (fp64 pose,
   double-float s), exact 1-NN of s_i, reject |s_i - t_j| > max_corr_dist, accumulate
   H = sum J^T J and g = sum J^T r for the chosen metric, solve H x = -g (6x6 Cholesky,
   fp64) and write pose_out = [exp([alpha]x) R, exp([alpha]x) t + tau].
   src [m*3] fp32; pose_in/pose_out fp64[16] device (may alias: in-place update);
   ws: device workspace (256-B aligned, >= cil_icp_workspace_bytes(m, params)).
   Optional outputs (NULL to skip): sys (device cil_icp_system), corr_idx[m] (int32
   original target index or -1 when rejected), corr_sqdist[m] (fp32 d^2 or +INF).
   On a degenerate system or zero correspondences pose_out = pose_in and sys->status
   says why. */
cil_status cil_icp_iterate(const cil_target* t, const float* src, int64_t m, const double* pose_in,
                           const cil_icp_params* params, void* ws, size_t ws_bytes, double* pose_out,
                           cil_icp_system* sys, int32_t* corr_idx, float* corr_sqdist,
                           cil_stream_t stream);

/* The ICP loop for params->max_iters iterations with no host round-trip:
   every iteration is enqueued up front; the pose and the stop flag live in device memory,
   so iterations after convergence, degeneracy or zero correspondences do no work.
   Correspondences use the certified warm start of SURVEY.md 8(a) row a2 in leaf form: a
   source point whose previous exact match j1 was found at anchor pose T_a, where every target
   outside j1's leaf L1 was at distance >= d_out, satisfies G = d_out - d1 > 2 |T p - T_a p|
   keeps L1 without a search (the nearest neighbour then provably lies in L1: for t not in
   L1, |s' - t| >= d_out - D > d1 + D >= |s' - t_j1|) and only L1's points are evaluated;
   every other point gets a full exact search (bounded by 1.1 max_corr_dist).  The result is
   identical to a full search every iteration up to exact d^2 ties.
   pose_init fp64[16] device; res: device cil_icp_result; iter_log (nullable) device
   fp64[max_iters*2] = {n_corr, rmse} per executed iteration (unexecuted rows are 0). */
cil_status cil_icp_run(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                       const cil_icp_params* params, void* ws, size_t ws_bytes, cil_icp_result* res,
                       double* iter_log, cil_stream_t stream);

/* The whole registration of one frame pair from HOST buffers (the end-to-end call: what the
   paper's benchmark times per pair, "Total registration times"): copies the
   target (and its normals), the source and the initial pose to the device, builds the index,
   runs cil_icp_run and copies the result back.  EVERY pointer is a HOST pointer here:
   target / normals fp32 [n*3] (normals NULL allowed for point-to-point), source fp32 [m*3],
   pose_init fp64[16] row-major (NULL = identity), result: host cil_icp_result.  Page-locked
   (pinned) host buffers make the copies asynchronous -- the source copy then runs on an
   internal second stream and overlaps the index build; pageable buffers work but are staged
   by the driver.  index: cil_index_params or NULL.  Device memory (inputs, workspace, result)
   comes from the library's stream-ordered pool and is released before returning.
   SYNCHRONOUS on `stream`: returns after the result is in *result (it synchronises that
   stream, not the device).  Errors as cil_target_build / cil_icp_run; on an error *result is
   not written.  Same kernels and bitwise the same result as the device-pointer calls. */
cil_status cil_icp_align_host(const float* target, const float* normals, int64_t n, const float* source, int64_t m,
                              const double* pose_init, const cil_icp_params* params, const cil_index_params* index,
                              cil_icp_result* result, cil_stream_t stream);

/* Surface normals of the TARGET points by PCA over their k nearest neighbours (SURVEY.md
   8(f) NEXT-3; "normal estimation", PAPER.md:172-176 10-NN normals oriented
   towards the viewpoint): for every target point p the exact k nearest targets (p itself
   included; equal distances order by the lowest original index), their mean and 1/k
   covariance (fp64), and the unit eigenvector of the smallest eigenvalue, flipped so that
   n . (view - p) >= 0.  k in [3, 16].  view: HOST double[3] (NULL = the origin).
   normals: device fp32 [n*3] in the target's original order; curvature (nullable): device
   fp32 [n] = lambda_min / trace.  The result can be passed to cil_target_build as the
   normals of a new target (the index itself is immutable).  Coordinates are expected to be
   finite; a point whose k-neighbourhood holds fewer than 3 finite neighbours (a non-finite
   point, or k-NN sets emptied by non-finite targets) gets a zero normal and curvature 0. */
cil_status cil_estimate_normals(const cil_target* t, int32_t k, const double* view, float* normals,
                                float* curvature, cil_stream_t stream);

/* ---- One ICP problem split across ranks ----
   The source is partitioned across GPUs (any split; each rank passes its own shard src[m] and
   its own workspace, the target is replicated).  Per iteration every rank calls
   cil_icp_shard_accumulate (certificates, exact 1-NN, reject, accumulate on its shard -- the
   steps of cil_icp_run) which writes its fp64 partial sums to sums[32] (device); the CALLER
   sums these 32 doubles across ranks (e.g. an NCCL all-reduce on the same stream), then every
   rank calls cil_icp_shard_finish with the reduced sums: the 6x6 solve and the pose update run
   redundantly and give bitwise identical poses on every rank (same inputs, same code).
   cil_icp_shard_begin sorts the shard and initialises the state (pose_init, iter_log as in
   cil_icp_run: global {n_corr, rmse} per iteration); cil_icp_shard_result copies the state to
   a device cil_icp_result.  Workspace: cil_icp_workspace_bytes(m).  Errors as cil_icp_run;
   m == 0 is allowed (an empty shard contributes zero sums). */
cil_status cil_icp_shard_begin(const cil_target* t, const float* src, int64_t m, const double* pose_init,
                               const cil_icp_params* params, void* ws, size_t ws_bytes, double* iter_log,
                               cil_stream_t stream);
cil_status cil_icp_shard_accumulate(const cil_target* t, const float* src, int64_t m, const cil_icp_params* params,
                                    void* ws, size_t ws_bytes, double* sums, cil_stream_t stream);
cil_status cil_icp_shard_finish(const cil_target* t, int64_t m, const cil_icp_params* params, void* ws,
                                size_t ws_bytes, const double* sums, double* iter_log, cil_stream_t stream);
cil_status cil_icp_shard_result(void* ws, cil_icp_result* res, cil_stream_t stream);

/* ---- Projective data association ----
   The paper's second correspondence engine: PAPER.md:83 ("different correspondence search
   engines (e.g., kd-tree based or projective)"), PAPER.md:140 ("one for correspondences by
   projective data association for the 3D case"); R23-R26.
   The target is an ORGANISED cloud: width*height points, packed fp32 xyz, row-major pixels
   (pixel (u, v) = point v*width + u) in the target camera frame; a pixel is invalid when its
   z <= 0 or a coordinate is not finite.  Source point p maps to s = R p + t (fp64) and
   projects to u = round(fx s_x / s_z + cx), v = round(fy s_y / s_z + cy), evaluated in fp64
   as ((f s) / s_z) + c and rounded half away from zero.  The pair
   (i, v*width + u) exists iff s_z > 0, 0 <= u < width, 0 <= v < height, the pixel is valid
   and |s - t| <= max_corr_dist (inclusive).  Steps a3-a7 are those of cil_icp_iterate.
   intrinsics: HOST struct, width, height >= 1, width*height <= INT32_MAX, fx, fy > 0 finite,
   cx, cy finite.  tgt / tgt_normals (nullable for point-to-point): device fp32 [w*h*3],
   caller-owned, read only (no index is built: the image IS the index).  The workspace is
   O(1) (cil_proj_workspace_bytes, independent of m); everything else as cil_icp_iterate /
   cil_icp_run (corr_idx = pixel index or -1). */
typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
} cil_intrinsics;

size_t cil_proj_workspace_bytes(int64_t m, const cil_icp_params* params);
cil_status cil_proj_iterate(const float* tgt, const float* tgt_normals, const cil_intrinsics* intrinsics,
                            const float* src, int64_t m, const double* pose_in, const cil_icp_params* params,
                            void* ws, size_t ws_bytes, double* pose_out, cil_icp_system* sys, int32_t* corr_idx,
                            float* corr_sqdist, cil_stream_t stream);
cil_status cil_proj_run(const float* tgt, const float* tgt_normals, const cil_intrinsics* intrinsics,
                        const float* src, int64_t m, const double* pose_init, const cil_icp_params* params,
                        void* ws, size_t ws_bytes, cil_icp_result* res, double* iter_log, cil_stream_t stream);

/* ---- Voxel-grid downsampling ----
   PAPER.md:125 ("general dimension grid-based point cloud downsampling"), PAPER.md:195 (the ICP
   benchmark's 1 cm voxel grid); R27-R29.  Point p falls in the bin
   k_a = floor((p_a - origin_a) / bin_size), evaluated in fp64.  One output point per non-empty
   bin: the fp64 mean of its points (summed in increasing input index) cast to fp32; output
   normals (nullable; need input normals): the fp64 mean of the bin's normals divided by its
   norm, or 0 if that norm < 1e-12.  Bins in ascending lexicographic (k_x, k_y, k_z) order.
   pts / normals: device fp32 [n*3]; origin: HOST double[3] (NULL = 0); out_pts / out_normals:
   device fp32 [n*3] (the worst case; the first *n_out rows are written); n_out: DEVICE int64,
   written stream-ordered (no host synchronisation) = the number of bins, or -1 when a key is
   not finite or an axis spans 2^21 bins or more.  n == 0 writes *n_out = 0.  Scratch ~44 B
   per point from the library's stream-ordered pool. */
cil_status cil_voxel_downsample(const float* pts, const float* normals, int64_t n, double bin_size,
                                const double* origin, float* out_pts, float* out_normals, int64_t* n_out,
                                cil_stream_t stream);

/* Static strings; cil_last_error is thread-local detail for the last failing call. */
const char* cil_status_string(cil_status s);
const char* cil_last_error(void);

/* Build/version info (static string). */
const char* cil_version(void);

/* Diagnostics: number of kernels this process has enqueued through the library so far
   (host counter, incremented at every launch). */
uint64_t cil_launch_count(void);

/* Diagnostics: per-launch CUDA-event timing.  While enabled, the library records a CUDA
   event pair on the launching stream around every cil_target_build call and every
   correspondence (K_nn), accumulation (K_acc) and nn_query launch.  cil_profile_read
   synchronises those events, adds their durations per class into *out and clears the list.
   Host-only API; not thread-safe. */
typedef struct {
    double build_ms, nn_ms, acc_ms, query_ms;   /* summed event durations */
    int64_t n_build, n_nn, n_acc, n_query;       /* number of timed launches */
    double sel_ms;                               /* certificate/selection kernel (cil_icp_run) */
    int64_t n_sel;
} cil_profile_stats;
cil_status cil_profile_enable(int on);
cil_status cil_profile_read(cil_profile_stats* out);

/* Diagnostics: bit 0 set = cil_icp_run does a full search every iteration (no certified
   warm start); used to measure the certificate.  Host-only, process-wide. */
cil_status cil_debug_set_flags(uint32_t flags);   /* bit 0 no certified warm start, bits 1-2 engine debug mode, bit 3 no point certificate, bit 4 caller order, bit 5 Morton order, bit 6 no small-problem brute-force path */

/* Tuning: the certificate skin of cil_icp_run.  A full search of point p uses the threshold
   (sqrt(best) + g)^2 with g = clamp(kappa * (p's displacement in the last iteration),
   min_frac * max_corr_dist, max_frac * max_corr_dist), so that its match is certified (leaf /
   candidate list) while p moves less than about g / 2 (a point moving faster than
   8 max_frac * max_corr_dist / kappa per iteration uses the minimum).  Defaults 0.001, 0.005, 16.
   0 <= min_frac <= max_frac <= 1, kappa >= 0.  Host-only, process-wide. */
cil_status cil_debug_set_cert_skin(double min_frac, double max_frac, double kappa);

/* Diagnostics: while buf (device int32, >= 16 per query slot) is non-NULL, every search-engine
   launch writes per processed query slot {flags, r, i0, i1, nF, best d2 after the packet
   phases, work items, final best d2, SM clocks of phases A, B, C, D+E, F, 0, 0, 0}.  NULL
   switches it off.  Host-only, process-wide.  Only a library built with -DCIL_TRACE=1 traces
   (the default build returns CIL_ERR_INVALID_ARG for a non-NULL buf). */
cil_status cil_debug_engine_trace(int32_t* buf);

/* Diagnostics: while buf (device uint64, 8 per iteration, filled with 0xff by the caller) is
   non-NULL, ICP launches write %globaltimer (ns) stamps of iteration it at buf[8*it + k]:
   k = 0 selection kernel start, 1 search kernel start, 2 accumulation (or projective) kernel
   start (each the earliest CTA), 3 the last CTA starts the final reduction, 4 solve/update
   done.  cil_icp_iterate / cil_proj_iterate use it = 0.  NULL switches it off.  Host-only,
   process-wide. */
cil_status cil_debug_timestamps(uint64_t* buf);

#ifdef __cplusplus
}
#endif
#endif /* CIL_H_ */
