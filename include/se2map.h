/*
 * se2map.h — C ABI of the B200-native SE(2) traversability library (libse2map.so).
 *
 * The library implements the data-parallel hot path of SEB-Naver's local mapping
 * (arXiv 2503.02412, §V): the robot-centric elevation window of Eq. 4
 * and Algorithm 1 evaluated for every SE(2) state
 * (x, y, yaw) of the window "in parallel", plus the incremental recompute of
 * the states whose footprint changed when the window moved.
 *
 * Conventions (readings R1-R21):
 *   - window cells: x = columns (fastest), y = rows; world cell I covers [I*r, (I+1)*r) (R6);
 *   - the window is [floor(x/r) - nx/2, ... + nx) x [floor(y/r) - ny/2, ... + ny) (Eq. 4, R6/R7);
 *   - yaw bin k has theta_k = -pi + 2*pi*k/n_yaw (R3); the footprint is the ellipse with
 *     semi-axes (e_x along x_yaw, e_y across) centred on the state (R2/R4), cell centres with
 *     q <= 1 + 1e-9 (R5), clipped to the window's known cells (R8/R9);
 *   - outputs per state: risk in [0,1] (Alg. 1 lines 10-18), signed pitch = asin(b3^T x_b) and
 *     roll = asin(b3^T y_b) (line 13, R13), z = fitted-plane height at the state centre (R14),
 *     traversable bit = no early return and not unknown (R17).  States with fewer than 3
 *     footprint cells or a degenerate covariance are "unknown": risk 1, trav 0, pitch/roll/z NaN.
 *
 * Ownership: the caller owns every pointer it passes; the library copies inputs before the
 * call returns (stream-ordered for device pointers) and retains nothing.  The library owns
 * all device memory it allocates (freed by se2m_destroy).
 * Concurrency: a handle has one owner and is not thread-safe; all work is ordered on the
 * handle's CUDA stream.  se2m_query / se2m_download synchronise that stream.
 * Errors: status codes only; no call aborts and no C++ exception crosses the ABI.  On
 * SE2M_ERR_INVALID_ARG the handle is unchanged.  se2m_last_error() gives a message.
 * Per-state degeneracy is not an error.
 */
#ifndef SE2MAP_H
#define SE2MAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct se2m_map se2m_map; /* opaque handle */

typedef enum {
  SE2M_OK = 0,
  SE2M_ERR_INVALID_ARG = 1,   /* bad dims / params / pointers (handle unchanged) */
  SE2M_ERR_OOM = 2,           /* device or host allocation failed */
  SE2M_ERR_CUDA = 3,          /* a CUDA runtime call or kernel launch failed */
  SE2M_ERR_UNSUPPORTED = 4,   /* parameter combination not built into this library */
  SE2M_ERR_OUT_OF_RANGE = 5,  /* a query / rectangle lies (partly) outside the window */
  SE2M_ERR_STATE = 6,         /* call order violated, e.g. assess before any elevation */
  SE2M_ERR_NCCL = 7           /* NCCL missing, communicator creation or a halo transfer failed */
} se2m_status;

enum { SE2M_FULL = 0, SE2M_INCREMENTAL = 1 };          /* se2m_assess_se2 mode */
enum { SE2M_MEM_HOST = 0, SE2M_MEM_DEVICE = 1 };       /* pointer kinds */
enum { SE2M_SHARD_NONE = 0, SE2M_SHARD_YAW = 1, SE2M_SHARD_ROWS = 2 };

typedef struct {
  int32_t nx, ny;          /* window cells, >= 1 each, nx*ny <= 2^31 */
  int32_t n_yaw;           /* yaw bins over [-pi, pi), >= 1 ("grids in SO(2)") */
  int32_t shard_mode;      /* SE2M_SHARD_*: which states this rank computes */
  double resolution;       /* l_res, m per cell, > 0 (Eq. 4; PAPER.md:248 uses 0.1) */
  double ellipse_ex;       /* footprint semi-axis along the heading, m, > 0 (Alg. 1 input e_x) */
  double ellipse_ey;       /* footprint semi-axis across the heading, m, > 0 (Alg. 1 input e_y) */
  double w_r[3];           /* risk weights w_r >= 0 (Alg. 1 input; default 0.4, 0.3, 0.3) */
  double kappa_max;        /* curvature limit > 0 (default 0.1) */
  double phi_x_max;        /* pitch limit, rad > 0 (0.52) */
  double phi_y_max;        /* roll limit, rad > 0 (0.52) */
  double robot_x, robot_y; /* initial robot position (m): window origin by Eq. 4 */
  int32_t rank, world_size;/* shard index / count (1 = single GPU) */
  int32_t device;          /* CUDA device ordinal */
  int32_t chain_segments;  /* yaw-chain segments S (0 = auto; see se2m_chain_segments); a tuning knob: changes FP32
                            * rounding only, results stay within the parity tolerances */
  void* cuda_stream;       /* cudaStream_t to order all work on, or NULL: the library creates one */
  /* NEXT-1 front-end (se2m_integrate_scan, readings R26-R30): */
  double fe_z_min, fe_z_max; /* body-frame height band of used points, m (default -1.5, 1.5) */
  double fe_gate;          /* Mahalanobis gate |z - h| / sqrt(s2 + s2_m) (default 2.0) */
  double fe_ray_eps;       /* ray-cast margin, m (default 0.05) */
  double fe_prior_var;     /* variance given to cells written by se2m_update_elevation, m^2 (default 1e-4) */
  /* NEXT-4 ("the GPU will compute the traversability ... using the inpainted elevation map"):
   * 0 = assess reads the map as it is (unknown cells are excluded from footprints, reading R9);
   * 1 = assess reads the nearest-neighbour inpainted view of the map (se2m_inpaint, reading R31),
   *     refreshed automatically when the map changed since the last refresh. */
  int32_t inpaint;
  int32_t step_graph;      /* 1: se2m_step submits its kernels (strip fill, edge and main assess) as ONE CUDA graph,
                            * re-captured every step and updated in place (cudaGraphExecUpdate), so the device runs them
                            * back to back; 0 (se2m_default_params): direct launches — on the 100 x 100 x 36 stream the
                            * graph measured 29.3 vs 28.9 us per step (the step is the assess kernel's latency, not
                            * launch gaps).  (inpaint = 1 maps always launch directly.) */
  /* Row-band halo transport (SE2M_SHARD_ROWS with world_size > 1, se2m_exchange_halo): the 128-byte NCCL
   * unique id every rank of the job passes (made by se2m_nccl_unique_id on one rank and sent to the others
   * by the caller's own bootstrap channel), or NULL for no communicator.  With an id, se2m_init creates the
   * library's NCCL communicator (rank, world_size) on `device` — a collective: every rank must call se2m_init
   * with the same id.  The library copies the id; the pointer need not outlive the call. */
  const void* nccl_unique_id;
} se2m_params;

/* NEXT-1: one LiDAR frame.  Rotations row-major (world <- body, body <- sensor), covariances 3x3. */
typedef struct {
  double R_B[9], p_B[3];   /* robot attitude and position (world) */
  double R_BS[9], p_BS[3]; /* LiDAR extrinsics: sensor -> body rotation, LiDAR position in the body frame */
  double Sigma_S[9];       /* sensor point noise */
  double Sigma_R[9];       /* attitude covariance, tangent space (right perturbation) */
  double Sigma_B[9];       /* position covariance */
} se2m_pose;

/* Fill *p with the defaults above (thresholds from PAPER.md:291 / SPEC S:300). */
void se2m_default_params(se2m_params* p);

/* Create a map: validates p, allocates the ring-buffered elevation window and output planes
 * on p->device, builds the per-yaw footprint tables.  All cells start unknown.
 * *out is set only on SE2M_OK. */
se2m_status se2m_init(const se2m_params* p, se2m_map** out);

/* Host-only (no device is touched): the share of the states the rank described by p computes.
 * Representative yaw bins [k_lo, k_hi) of n_rep (bin k + n_rep shares bin k's footprint when n_yaw is
 * even); world tile rows TJ (of tile_y cells) with TJ mod row_mod == row_rank.  Any pointer may be NULL. */
se2m_status se2m_shard_plan(const se2m_params* p, int32_t* n_rep, int32_t* k_lo, int32_t* k_hi,
                            int32_t* tile_y, int32_t* row_mod, int32_t* row_rank);

/* Free everything (synchronises the stream).  NULL-safe. */
void se2m_destroy(se2m_map* m);

/* Write elevations for the window-local rectangle [i0, i0+w) x [j0, j0+h) (columns x rows),
 * the inpainted map M of Alg. 1.  heights: row-major, leading dimension
 * ld >= w floats; known: same layout in bytes (1 = known), or NULL = all known.  mem says
 * whether both pointers are host or device memory.  The rectangle must lie inside the window
 * (else SE2M_ERR_OUT_OF_RANGE, nothing written).  Marks the rectangle dirty for INCREMENTAL. */
se2m_status se2m_update_elevation(se2m_map* m, int32_t i0, int32_t j0, int32_t w, int32_t h,
                                  const float* heights, int64_t ld, const uint8_t* known,
                                  int32_t mem);

/* Eq. 4: recentre the window on the robot at (robot_x, robot_y): the new
 * origin is floor(x/r) - nx/2 (IEEE double, reading R7); cells that leave the window become
 * unknown ("removed in parallel").  No data moves (ring buffer).  Returns the
 * origin displacement in cells through out_di / out_dj (either may be NULL).  Marks the
 * exposed and the vacated strips dirty.  State records (se2m_query / se2m_download) of cells that
 * entered the window are undefined until the next se2m_assess_se2; the SDF must be recomputed. */
se2m_status se2m_shift_window(se2m_map* m, double robot_x, double robot_y, int32_t* out_di,
                              int32_t* out_dj);

/* Algorithm 1 for every SE(2) state of this rank's share (mode SE2M_FULL), or
 * only for the states whose footprint touches a cell changed since the last assess
 * (SE2M_INCREMENTAL; results are bit-identical to FULL).  Asynchronous on the handle's stream: the
 * tiles at the window's left / right edge run in a second kernel on an internal stream that is
 * forked from and joined back into the handle's stream with events, so work queued on the handle's
 * stream after this call (and se2m_synchronize) sees all results.  SE2M_ERR_STATE if no elevation
 * was ever written; SE2M_ERR_UNSUPPORTED if a footprint's tables cannot fit a CTA's shared memory. */
se2m_status se2m_assess_se2(se2m_map* m, int32_t mode);

/* One rolling-window step against a larger device-resident source map, H1 + H2 + H9 in one call (two
 * kernel launches): recentre on (x, y) as se2m_shift_window (Eq. 4), write the cells
 * that entered the window from `world` — a device plane of heights covering world cells
 * [world_I0, world_I0 + world_w) x [world_J0, world_J0 + world_h), leading dimension world_ld
 * (elements), NaN = unknown; window cells outside it become unknown — and assess INCREMENTAL.
 * mem must be SE2M_MEM_DEVICE.  Same results as shift_window + update_elevation(strips) +
 * assess_se2(INCREMENTAL), bit for bit.  Optional out_di / out_dj as in se2m_shift_window. */
se2m_status se2m_step(se2m_map* m, double x, double y, const float* world, int64_t world_ld,
                      int64_t world_I0, int64_t world_J0, int32_t world_w, int32_t world_h, int32_t mem,
                      int32_t* out_di, int32_t* out_dj);

/* n world-frame queries xyt[3*q + {0,1,2}] = (x, y, theta): the state of the window cell
 * containing (x, y) at the nearest yaw bin (reading R3/R6).  Any output pointer may be NULL;
 * outputs are host memory of n entries.  Entries outside the window (or of yaw bins this
 * rank does not own) get NaN / trav 0 and the call returns SE2M_ERR_OUT_OF_RANGE after
 * filling all others.  Synchronises the stream. */
se2m_status se2m_query(se2m_map* m, int64_t n, const double* xyt, float* risk, float* pitch,
                       float* roll, float* z, uint8_t* trav);

/* Asynchronous query (the planner's pipelined read): the same lookups as se2m_query, written to
 * out = 5 x n floats, planar: risk[n], pitch[n], roll[n], z[n], trav[n] (1.0 / 0.0); states outside the
 * window (or not owned) give NaN / risk 1 / trav 0.  xyt and out are host (mem = SE2M_MEM_HOST) or device
 * pointers.  Pinned (page-locked) host buffers are read and written in place by the query kernel (zero copy);
 * pageable ones are staged through device memory with copies on the stream.  Queued on the map's stream and not
 * synchronised: out is valid after se2m_synchronize (or an event recorded on the stream); xyt must stay
 * untouched until then.  No out-of-range status (read the NaNs). */
se2m_status se2m_query_async(se2m_map* m, int64_t n, const double* xyt, float* out, int32_t mem);

/* Whole output planes in LOGICAL window order, layout [k][j][i] (n_yaw * ny * nx entries per
 * non-NULL pointer; trav as bytes 0/1).  mem says whether the output pointers are host or
 * device memory.  States this rank does not own (yaw bins or tile-row bands, see se2m_shard_plan) are
 * NaN / 0 (compact downloads: risk 1.0 / trav 0).  Synchronises. */
se2m_status se2m_download(se2m_map* m, float* risk, float* pitch, float* roll, float* z,
                          uint8_t* trav, int32_t mem);

/* Compact copy of the map for planners (the paper sends the risk map to the CPU):
 * risk_h[k][j][i] = the IEEE-754 binary16 bit pattern of risk (round to nearest even; relative error
 * <= 2^-12 for risk >= 2^-14 and absolute <= 2^-25 below, so within the parity tolerance 1e-3 |risk| + 1e-6 of
 * the FP32 state everywhere on [0, 1]; unknown / not owned = 1.0) and the traversable bits re-packed in
 * logical order, trav_bits[k][j][w] bit b = column 32 w + b (ceil(nx/32) words per row, bits past nx zero).
 * Either pointer may be NULL; mem as in se2m_download.  Synchronises.  (pitch, roll and z stay on the device:
 * se2m_query / se2m_download.) */
se2m_status se2m_download_compact(se2m_map* m, uint16_t* risk_h, uint32_t* trav_bits, int32_t mem);

/* The same compact map without its redundant half: Risk and traversability are pi-periodic in theta
 * (bins k and k + n_yaw/2 have the same footprint and pitch / roll of opposite sign, and Alg. 1 uses only
 * their absolute values: PAPER.md:145-151, readings R13 / R23), so for even n_yaw only the n_rep =
 * n_yaw / 2 representative planes are written — plane k serves bins k and k + n_rep — with the layout of
 * se2m_download_compact (n_rep instead of n_yaw planes; odd n_yaw: all planes).  Host destinations are
 * filled ASYNCHRONOUSLY from double-buffered device staging on the map's copy stream, so the transfer
 * overlaps the next update / assess; the buffers may be read after se2m_synchronize.  Device
 * destinations are written on the map's stream. */
se2m_status se2m_download_compact_rep(se2m_map* m, uint16_t* risk_h, uint32_t* trav_bits, int32_t mem);
/* (With row-band sharding, se2m_download_compact_rep writes only the rank's own logical rows, packed in
 * increasing order: planes of n_rows rows.)  The rank's own logical rows of the current window
 * (all ny rows unless row-band sharded): *n of them, listed in rows[] if rows is not NULL. */
se2m_status se2m_owned_rows(const se2m_map* m, int32_t* rows, int32_t* n);

/* Row-band halo exchange (SE2M_SHARD_ROWS, world_size G > 1; SURVEY.md §8(e) "row bands + halo";
 * a state's risk reads the elevation under its footprint, up to R cells away).  Rank g owns
 * the world tile rows TJ = g (mod G) (se2m_shard_plan).  A rank whose update_elevation wrote only its own
 * rows (se2m_owned_rows) lacks the R_T rows on either side of each owned tile row, which rank g - 1 and
 * rank g + 1 own.  Exchange, per step, before se2m_assess_se2:
 *   se2m_halo_pack(m, -1, a)  -> send a to rank g - 1;   se2m_halo_pack(m, +1, b) -> send b to rank g + 1;
 *   receive c from rank g + 1 -> se2m_halo_unpack(m, +1, c);  d from rank g - 1 -> se2m_halo_unpack(m, -1, d).
 * se2m_exchange_halo does all of it inside the library over NCCL (below); pack / unpack stay public for
 * callers with their own transport.  Buffers: device memory of cap x slab_rows x nx
 * floats (se2m_halo_size), slab q = slab_rows window-width rows in logical column order; rows outside the
 * window are NaN in a packed buffer and ignored on unpack.  Slab lists are derived from the window origin,
 * which every rank shares, so sender and receiver agree without metadata.  pack only reads the ring;
 * unpack writes the received rows and marks them dirty (INCREMENTAL).  Both are asynchronous on the map's
 * stream.  SE2M_ERR_INVALID_ARG unless row-sharded with world_size > 1 (or dir / pointers bad);
 * SE2M_ERR_UNSUPPORTED when R_T exceeds the tile height (the halo would reach tile rows TJ +- 2). */
se2m_status se2m_halo_size(const se2m_map* m, int32_t* cap, int32_t* slab_rows);
se2m_status se2m_halo_pack(se2m_map* m, int32_t dir, float* dst);
se2m_status se2m_halo_unpack(se2m_map* m, int32_t from, const float* src);
/* The exchange itself, inside the library ("ncclSend/Recv to (g +- 1) mod G"): packs this
 * rank's outgoing slabs (as se2m_halo_pack, both directions), runs ncclGroupStart; ncclSend(first rows ->
 * g - 1); ncclRecv(<- g + 1); ncclSend(last rows -> g + 1); ncclRecv(<- g - 1); ncclGroupEnd on the map's
 * stream over the communicator made by se2m_init from params.nccl_unique_id, and unpacks what arrived (as
 * se2m_halo_unpack from both sides).  Every rank calls it once per step after writing its own rows and before
 * se2m_assess_se2; all of it is asynchronous on the map's stream (no host synchronisation).  With G = 2 both
 * neighbours are the same peer: sends and receives between a pair match in issue order, and the order above
 * pairs each send with the peer's receive of the same slab set.  SE2M_ERR_INVALID_ARG unless row-sharded with
 * world_size > 1; SE2M_ERR_STATE without a communicator; SE2M_ERR_NCCL when a transfer fails to enqueue.
 * Device buffers (4 x cap x slab_rows x nx floats) are allocated on first use. */
se2m_status se2m_exchange_halo(se2m_map* m);
/* Host-only: a fresh NCCL unique id (out, bytes >= 128) for params.nccl_unique_id; SE2M_ERR_NCCL when NCCL
 * cannot be loaded.  *version (may be NULL) = the loaded NCCL's version code (e.g. 22809). */
se2m_status se2m_nccl_unique_id(void* out, int32_t bytes, int32_t* version);
/* Diagnostic (the calls se2m_exchange_halo makes, on hardware with one GPU): a one-rank NCCL communicator on
 * `device` (ncclGetUniqueId, ncclCommInitRank), one grouped ncclSend + ncclRecv of `count` floats from a
 * device buffer to a second one on the same rank (ncclGroupStart / End on a private stream), the received
 * floats compared with the sent ones on the host, ncclCommDestroy.  *version (may be NULL) = the loaded NCCL's
 * version code.  SE2M_OK when the data arrived intact; SE2M_ERR_NCCL (NCCL missing, a call failed, or the data
 * differ), SE2M_ERR_CUDA, SE2M_ERR_INVALID_ARG (count < 1).  Synchronous; leaves the current device as it was. */
se2m_status se2m_nccl_selftest(int32_t device, int64_t count, int32_t* version);

/* Host-only (no device): the slab list of rank `sender` for window origin row J_M: first_rows[q] = first
 * world row of slab q (slab_rows rows), or INT64_MIN past the end of the list; last = 0: the first rows of
 * the sender's tile rows (the slabs it sends to rank sender - 1), 1: the last rows (to sender + 1).
 * first_rows (cap entries) may be NULL to query cap / slab_rows. */
se2m_status se2m_halo_plan(const se2m_params* p, int64_t J_M, int32_t sender, int32_t last, int32_t* cap,
                           int32_t* slab_rows, int64_t* first_rows);

/* NEXT-1: integrate one LiDAR frame into the elevation window (§V.A, Fig. 3):
 * points (n x 3 float, sensor frame; host or device per mem) are transformed with the pose, points
 * outside the window or outside the body-frame height band are ignored, each point gets the
 * height variance of P:113-120; then every ray (LiDAR -> used point) resets to unknown the cells it
 * crosses whose height exceeds the ray's highest height over the cell + fe_ray_eps (the
 * point's own cell excluded), and the points are fused per cell in input order by a 1-D Kalman filter
 * with the Mahalanobis gate / higher-wins rule.  FP64 arithmetic in a fixed order; cells
 * keep float32 height and variance.  Marks the touched cells dirty.  Optional out_counts[5] = points
 * used, outside the map, outside the band, with sigma^2 <= 0, and ray-reset events.  Synchronises. */
se2m_status se2m_integrate_scan(se2m_map* m, const float* points, int64_t n, const se2m_pose* pose,
                                int32_t mem, int64_t* out_counts);

/* Heights and variances of the window in logical order (ny x nx each, NaN height = unknown). */
se2m_status se2m_download_elevation(se2m_map* m, float* heights, float* variances, int32_t mem);

/* NEXT-4: nearest-neighbour inpainting ("can be inpainted by classical methods", PAPER.md:248
 * "Both methods utilize nearest-neighbor interpolation for elevation inpainting").  Reading R31: every
 * unknown cell of the window takes the height of its nearest known cell of the window (Euclidean distance
 * on grid indices; ties to the known cell first in row-major (j, i) order); known cells keep theirs.  The
 * result is a separate view: the map itself (the Kalman state) keeps its unknown cells.  Cells whose view
 * value changed are marked dirty for INCREMENTAL assessment.  SE2M_ERR_STATE when no cell of the window
 * is known (the view is then all unknown).  Synchronises (reads back a counter and a bounding box). */
se2m_status se2m_inpaint(se2m_map* m);

/* The inpainted view in logical order (ny x nx; refreshed first if the map changed). */
se2m_status se2m_download_inpainted(se2m_map* m, float* heights, int32_t mem);

/* NEXT-2: signed distance field of the explicit obstacles (Risk = 1) of
 * every yaw layer, from the last assess ("the corresponding signed distance field (SDF)
 * will be generated"; "the distance to the edge of the nearest region, with negative
 * values inside obstacles").  Reading R24: a free state's value is the Euclidean distance in metres
 * between cell centres to the nearest obstacle state of the same layer, an obstacle state's value is
 * minus the distance to the nearest free state; cells outside the window are neither; values are
 * clamped to [-d_max, d_max] (d_max / resolution <= 96).  Exact within d_max.  Asynchronous.
 * Bins k and k + n/2 share an obstacle set and thus a layer.  SE2M_ERR_UNSUPPORTED with row sharding;
 * SE2M_ERR_STATE when the risk map is stale (no assess since the last shift / update / scan).  With yaw
 * sharding only the owned layers are computed: the others read as NaN. */
se2m_status se2m_compute_sdf(se2m_map* m, double d_max);

/* The SDF in logical order, out[k][j][i] for all n_yaw bins (mem: host or device).  Synchronises. */
se2m_status se2m_download_sdf(se2m_map* m, float* out, int32_t mem);

/* Stand-alone SDF of obstacle masks (no map): mask[layer][j][i] bytes (1 obstacle, 0 free), logical
 * order, out the same layout in float metres; same definition as se2m_compute_sdf.  mem: whether mask
 * and out are host or device memory.  Runs on `device`, synchronous. */
se2m_status se2m_sdf_from_mask(const uint8_t* mask, int32_t nx, int32_t ny, int32_t layers,
                               double resolution, double d_max, float* out, int32_t mem, int32_t device);

/* NEXT-3: the planner's map access: trilinear interpolation over (x, y, theta) of
 * field 0 = Risk or 1 = SDF (after se2m_compute_sdf), theta cyclic across +-pi; value[q] and the exact
 * gradient of the interpolant grad[3q..3q+2] = (d/dx, d/dy, d/dtheta) per metre / radian.  Lattice:
 * node (i, j, k) at ((I_M + i + 1/2) r, (J_M + j + 1/2) r, theta_k).  Queries whose 8 corner nodes are
 * not all inside the window (or owned) give NaN and the call returns SE2M_ERR_OUT_OF_RANGE after
 * filling the others.  Any output pointer may be NULL (host memory).  Synchronises. */
se2m_status se2m_query_trilinear(se2m_map* m, int64_t n, const double* xyt, int32_t field, float* value,
                                 float* grad);

/* Asynchronous form (the planner's pipelined access): the same interpolation written to out = 4 x n floats,
 * planar: value[n], d/dx[n], d/dy[n], d/dtheta[n] (NaN where a corner is outside / not owned).  xyt and out
 * are host or device pointers per mem (pinned host buffers are read and written in place by the kernel, pageable
 * ones staged); queued on the map's stream, not
 * synchronised (out valid after se2m_synchronize; xyt untouched until then). */
se2m_status se2m_query_trilinear_async(se2m_map* m, int64_t n, const double* xyt, int32_t field, float* out,
                                       int32_t mem);

/* Window origin (world cell of logical (0,0)) and the owned representative-yaw range. */
se2m_status se2m_get_origin(const se2m_map* m, int64_t* I_M, int64_t* J_M);

/* Number of footprint cells |P_k| for yaw bin k (0 <= k < n_yaw) and the stencil radius R. */
se2m_status se2m_stencil_info(const se2m_map* m, int32_t k, int32_t* n_cells, int32_t* radius);

/* Yaw-chain segments of the map: the representative bins [0, H) are cut into S segments at the
 * bounds floor(H s / S); moments are carried from bin k-1 to bin k inside a segment and recomputed from whole
 * footprint rows at each bound; S = H: no chain (small maps).  A state's FP32 rounding depends on S, never on
 * sharding: a yaw shard (se2m_shard_plan: the balanced split [H g / G, H (g + 1) / G) of the representative bins)
 * that does not start on a bound replays the chain from its segment's bound without storing, so yaw-sharded
 * maps equal the unsharded one bit for bit (with no replay when G divides S). */
se2m_status se2m_chain_segments(const se2m_map* m, int32_t* segments);

/* World-aligned tile of states one CTA assesses: TX columns x TY rows (SE2M_SHARD_ROWS gives world
 * tile row TJ = floor(J / TY) to rank TJ mod world_size). */
se2m_status se2m_tile_info(const se2m_map* m, int32_t* tile_x, int32_t* tile_y);

/* Block until all work queued on the handle's streams (its stream and its copy stream) is done. */
se2m_status se2m_synchronize(se2m_map* m);

/* Diagnostics (debug builds compiled with SE2M_PHASES, tools/build_phases.sh; SE2M_ERR_UNSUPPORTED otherwise):
 * per-warp records of the assess kernels' phase boundaries (%globaltimer ns: start, halo in shared memory, tile
 * plane, prefix planes and tables, states done, end; then blockIdx.x, blockIdx.y, kernel mode, flags), 64 bytes
 * each, copied into out (host memory, up to max_records); *n = records written since the last reset (process-
 * wide, all handles).  reset != 0 restarts the count.  Synchronises the stream. */
se2m_status se2m_debug_phases(se2m_map* m, void* out, int64_t max_records, int32_t reset, int64_t* n);

/* Kernel launches issued by this handle since creation (for the bench's gpu_launches). */
int64_t se2m_launch_count(const se2m_map* m);

/* Per-handle message for the last failing call; valid until the next call on m.
 * se2m_last_error(NULL) returns the message of the last failed se2m_init. */
const char* se2m_last_error(const se2m_map* m);

#ifdef __cplusplus
}
#endif
#endif /* SE2MAP_H */
