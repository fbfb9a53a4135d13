// se2m_internal.h — shared between the C-ABI runtime (se2map.cu) and the kernels (assess.cu).
// Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace se2m {

// Spatial tile of states handled by one CTA: world-aligned, TX = one warp wide,
// tile_rows(R_T) rows (32 for R_T <= 12, else 16, to fit >= 2 CTAs per SM in shared memory).
constexpr int TX = 32;
// threads per assess CTA: 256 (8 warps, 2 CTAs per SM) — except R_T = 16 (the 0.05 m high-res footprint): one
// CTA of 512 threads (16 warps) per SM on 32-row tiles, because its tile planes leave shared memory for only
// one CTA per SM and 8 warps cannot hide the latency of the chain loops
#ifndef SE2M_R16_THREADS
#define SE2M_R16_THREADS 512
#endif
constexpr int nthreads(int R_T) { return (R_T > 12 && R_T <= 16) ? SE2M_R16_THREADS : 256; }
#ifndef SE2M_TY_SMALL
#define SE2M_TY_SMALL 32
#endif
constexpr int tile_rows(int R_T) { return R_T <= 12 ? SE2M_TY_SMALL : (nthreads(R_T) == 512 ? 32 : 16); }
// shared-memory layout choice of the assess kernel: up to R_T = 24 the h^ plane is separate and border
// tiles also run on the yaw chain (both run tables in shared memory); at R_T = 32 the plane aliases the
// validity prefixes (interior tiles only) and border tiles take the full rows of every bin
constexpr bool chain_border(int R_T) { return R_T <= 24; }

// Stencil radii the assess kernel is instantiated for (R_T >= the footprint radius R).
constexpr int kRadii[] = {4, 8, 12, 16, 24, 32};
constexpr int kMaxRects = 8;  // dirty rectangles passed by value to an INCREMENTAL launch

struct AssessParams {
  // window / ring buffer: world cell (I, J) lives at physical (I mod nx, J mod ny)
  int nx, ny;            // window == ring dims
  int ldh;               // heights row pitch in floats (multiple of 4: 16-B TMA stride)
  long long I_M, J_M;    // window origin, world cells (Eq. 4)
  const float* h;        // [ny][ldh] physical, NaN = unknown
  int pxM, pyM;          // physical column / row of logical (0, 0) = I_M mod nx, J_M mod ny
  // outputs: state records [k][ny][nx] float4 (risk, pitch, roll, z), physical (ring) layout;
  // traversable bits [k][ny][trav_words], word = floor(I/32) mod trav_words, bit = I mod 32 (world I)
  float4* out;
  uint32_t* trav;
  int trav_words;        // ceil(nx/32) + 1: the window's 32-groups map to distinct words
  // yaw: rep bins k in [0, H); bin k + H (if paired) is the same footprint, x_yaw negated
  int n_yaw, H, paired;
  int R;                 // true footprint radius (cells); kernel template R_T >= R
  // Stencil tables as "run entries" (e_minus, e_plus, d, 0): a run sum is P[e_plus] - P[e_minus] of halo
  // row d (= dj + R_T), element offsets relative to the state's own prefix column.  full: the non-empty
  // rows of bin k; chain: the full rows when k % period == 0, else the endpoint corrections from bin
  // k-1 to bin k (moments carried along the yaw chain).  Entries of bin k: [off[k], off[k+1]).
  const int4* full;
  const int4* full_fmt;  // the same full rows in the kernel's entry format (8 e-, 8 e+, 4 e-, float dj)
  const int* full_off;   // [H+1]
  // chain (interior tiles) is stored in the kernel's shared-memory format: per bin first the prefix
  // entries (8 e_minus, 8 e_plus, 4 e_minus, float dj) — byte offsets into {P0, P2} and PX — then, from
  // chain_mid[k], single-cell entries (4 e, float sgn, float sgn di, float sgn dj): a cell that enters
  // (sgn = +1) or leaves (-1) the footprint between bins k-1 and k, e = its element offset into the h^
  // plane (stride PW, like the prefix rows).  Endpoint moves of <= 2 cells (nearly all at 5-degree bins)
  // become cell entries (one 4-byte load per state instead of four prefix loads).
  const int4* chain;
  const int* chain_off;  // [H+1]
  const int* chain_mid;  // [H]
  // yaw chain in S = seg segments: bin k restarts the chain (moments from whole footprint rows) iff k is a
  // segment bound floor(H s / S) (seg_bound); S = H: no chain.  A CTA takes seg_chunk consecutive segments
  // (its chunk): blockIdx.y covers segments [s0 + c y, s0 + c (y + 1)), s0 = the segment of k_begin.
  int seg, seg_chunk, n_chunks;
  int seg_first;                // the segment of k_begin
  const int* segb;              // [seg + 1] segment bounds seg_bound(s)
  const unsigned char* seg_rst; // [H] 1 where a bin is a segment bound (chain restart)
  int tab_cap;           // max entries of one CTA's chunk (shared-memory table size)
  const float4* geo;     // [H] full-stencil (N, Sxx, Sxy, Syy) in cell units (Sx = Sy = 0)
  const float4* geoc;    // [H][4] full-stencil geometry for interior tiles (see assess.cu, arrow2), metres
  const float2* cs;      // [H] (cos, sin) of theta_k, k < H (reading R3)
  float r;               // resolution (m)
  // risk (Alg. 1 lines 10-18), all float
  float kappa_max, phi_x_max, phi_y_max;
  float wk, wx, wy;      // w_r[0]/kappa_max, w_r[1]/phi_x_max, w_r[2]/phi_y_max
  // tiles: world tile (TI, TJ) covers I in [TI*TX, TI*TX+TX), J in [TJ*TY, TJ*TY+TY), TY = tile_rows(R_T)
  // CTA b runs world tile (TI0 + b % tiles_x, TJ0 + row_first + (b / tiles_x) * row_mod): row_mod > 1
  // shards tile rows across ranks (SE2M_SHARD_ROWS); n_rects > 0 restricts the launch to the tiles
  // inside rects (INCREMENTAL), [x0, x1) x [y0, y1) in tiles relative to (TI0, TJ0).
  long long TI0, TJ0;
  int tiles_x;
  int row_first, row_mod;
  // downloads: row-band ownership of this rank (SE2M_SHARD_ROWS): logical row j is owned iff
  // (floor((J_M + j) / own_ty) - own_rank) mod own_G == 0 (own_G = 1: every row)
  int own_G, own_rank, own_ty;
  int n_rects;
  int4 rects[kMaxRects];
  int k_begin, k_end;    // representative-bin range this launch covers (k_begin: a yaw-chain restart)
  int k_store;           // first bin stored: bins [k_begin, k_store) only replay the yaw chain (a yaw shard
                         // whose first bin lies inside a chain period carries the moments from the period's
                         // restart, so its states are bit-identical to the unsharded map's)
  int k_chunk;           // rep bins per CTA (grid.y = ceil((k_end-k_begin)/k_chunk))
  // vertical-window-edge tiles (tile columns tcols[0 .. n_tcols) of the launch) run in a second kernel,
  // assess_kernel<R_T, 1>, on the edge stream (tsplit = 1); the main launch skips them
  int tsplit, n_tcols;
  int tcols[4];
  int main_first;        // (host) launch the main kernel before the edge kernel: set when both grids fit one wave
                         // together, so neither waits for slots and the main kernel's longer CTAs start first
  int use_tma;           // tensor map valid
  int force_general;     // some full stencil is degenerate (< 3 cells or collinear): no interior fast path
};

// Yaw-chain segments (AssessParams::seg): segment s covers representative bins [seg_bound(s), seg_bound(s + 1)).
// With S <= H every segment holds >= 1 bin; the balanced yaw shards of se2m_shard_plan, [H g / G, H (g + 1) / G),
// start on segment bounds whenever G divides S (a shard starting elsewhere replays from its segment's bound).
// (host side; the kernels read the bounds and restart flags from tables built from these)
inline int seg_bound(int H, int S, int s) { return (int)((long long)H * s / S); }
inline int seg_of(int H, int S, int k) {
  int s = (int)((long long)k * S / H);
  if (s + 1 <= S && seg_bound(H, S, s + 1) <= k) ++s;  // (at most one step: segments hold >= 1 bin)
  return s;
}
inline bool seg_restart(int H, int S, int k) { return seg_bound(H, S, seg_of(H, S, k)) == k; }

// Launch the assess kernel (one CTA per (tile, yaw chunk)).  Returns cudaSuccess or the launch error.
// dynamic shared memory of one assess CTA (halo, prefix planes, h^ plane, run tables of tab_cap entries)
size_t assess_smem_bytes(int R_T, int tab_cap, int k_chunk);
// resident CTAs per SM of the main assess kernel at that dynamic shared memory (occupancy API; 0 on error)
int assess_ctas_per_sm(int R_T, size_t smem);
// With p.tsplit the edge-tile kernel runs on `edge` (forked from / joined into `stream` with the two
// events); *n_launch = kernels launched.
// pe: the edge kernel's parameters (its own yaw-chain tables and chunking; otherwise p's).  side[0 .. n_side):
// extra launches of the main kernel on the edge stream (the window's top / bottom border tile rows, with the
// edge chain), side_tiles[q] tiles each; the main launch p covers the other n_tiles - sum(side_tiles) tiles.
cudaError_t launch_assess(const AssessParams& p, const AssessParams& pe, int R_T, int n_tiles, const AssessParams* side,
                          const int* side_tiles, int n_side, const CUtensorMap* tmap, cudaStream_t stream,
                          cudaStream_t edge, cudaEvent_t fork, cudaEvent_t join, int* n_launch);

// SE2M_PHASES debug builds: per-warp phase timestamps of the assess kernel (PhaseRec in assess.cu: 6 x u64 + 4 x i32)
cudaError_t debug_phases(void* out, long long max_records, int reset, long long* n, cudaStream_t s);

// Small helpers (same file as the kernels).
// se2m_step: the window cells that entered (up to 2 logical rectangles (i0, j0, w, h)) from a device
// plane of world heights covering [wI0, wI0 + ww) x [wJ0, wJ0 + wh) (NaN = unknown; outside: unknown)
struct FillArgs {
  float* h;
  float* var;
  float prior_var;
  int ldh, nx, ny, pxM, pyM;
  long long I_M, J_M;
  const float* world;
  long long world_ld, wI0, wJ0;
  int ww, wh;
  int n;
  int4 rect[2];
};
cudaError_t launch_fill_strips(const FillArgs& f, cudaStream_t s);
cudaError_t launch_clear_rect(float* h, int ldh, int x0, int y0, int w, int hgt, int nx, int ny,
                              cudaStream_t s);
cudaError_t launch_scatter_rect(float* h, float* var, float prior_var, int ldh, int nx, int ny, int px0, int py0,
                                int w, int hgt, const float* src, long long ld, const uint8_t* known, cudaStream_t s);
// Row-band halo slabs (SE2M_SHARD_ROWS; enumeration in se2map.cu): slab q holds world rows
// [W_q, W_q + R_T), W_q = TJ_q TY (the first rows of tile row TJ_q) or TJ_q TY + TY - R_T (the last rows),
// TJ_q = TJ0 + q G while TJ_q <= TJb; buffer layout [q][r][i], i = logical column.  Rows outside the
// window: NaN in a packed buffer, untouched in the ring on unpack.
struct HaloArgs {
  float* h;                // ring heights [ny][ldh]
  float* buf;              // device slabs [cap][R_T][nx]
  int ldh, nx, ny, pxM, pyM;
  long long J_M;           // window origin row (world)
  long long TJ0, TJb;      // first tile row of the list, last tile row of the range
  int G, TY, R_T, last;    // last = 1: the last R_T rows of each tile row, 0: the first R_T rows
  int unpack;              // 0: ring -> buf, 1: buf -> ring
};
cudaError_t launch_halo(const HaloArgs& a, int cap, cudaStream_t s);
cudaError_t launch_gather_logical(const AssessParams& p, int k_lo, int k_hi, float* risk,
                                  float* pitch, float* roll, float* z, uint8_t* trav, cudaStream_t s);
// packed_rows > 0: only the rank's own rows (row-band sharding), packed in increasing order
cudaError_t launch_gather_compact(const AssessParams& p, int k_lo, int k_hi, uint16_t* risk_h, uint32_t* bits,
                                  int words_per_row, cudaStream_t s, int packed_rows = 0);
// World (x, y, theta) -> ring indices, resolved on the device in FP64 exactly as readings R3/R6 state.
struct QueryGeo {
  double r, dth;
  long long I_M, J_M;
  int nx, ny, n_yaw, H, paired;
  int k_lo, k_hi;          // owned representative bins
  int row_mod, row_rank;   // owned world tile rows (TJ mod row_mod == row_rank)
  int TY, trav_words;
};
// nearest state (H10): out 5 x n (risk, pitch, roll, z, trav); *n_out += queries outside / not owned
cudaError_t launch_query(const AssessParams& p, const QueryGeo& g, int n, const double* xyt, float* out, int* n_out,
                         cudaStream_t s);

// ---- NEXT-1: elevation front-end (frontend.cu) -----------------------------------------------------
struct FePose {
  double R_B[9], p_B[3], R_BS[9], p_BS[3], Sigma_S[9], Sigma_R[9], Sigma_B[9];  // row-major 3x3
};
struct FrontendArgs {
  FePose pose;
  double r, z_min, z_max, gate, ray_eps;
  double sx, sy, sz;     // LiDAR position in the world, R_B p_BS + p_B (host, fixed order)
  long long I_M, J_M;
  int nx, ny, ldh, pxM, pyM;
  int key_bits;          // radix-sort key width: ring cell indices < 2^key_bits - 1
  int key_none;          // 2^key_bits - 1: the key of a filtered point (sorts last)
};
struct FrontendScratch {
  int *key, *idx, *skey, *sidx;
  double4* meas;         // (x, y, z_l, sigma^2) per point
  int* counts;           // [5]: used, outside the map, outside the height band, bad variance, ray resets
  int* bbox;             // [4]: logical i_min, i_max, j_min, j_max of the cells touched
  void* temp;
  size_t temp_bytes;
  size_t cap;
};
cudaError_t frontend_run(const FrontendArgs& a, int n, const float* pts, FrontendScratch& s, float* h, float* var,
                         cudaStream_t st);
size_t frontend_temp_bytes(int n);

// ---- NEXT-2: signed distance field of the Risk = 1 set per yaw layer (sdf.cu) ----------------------
struct SdfParams {
  int nx, ny, layers;    // logical window size, number of layers
  float r, d_max;        // resolution, clamp (m)
  int W;                 // search radius in cells = ceil(d_max / r)
  // input: map mode (trav != nullptr): obstacle = traversable bit 0 of the map's state at logical (i, j)
  const uint32_t* trav;
  int trav_words, pxM, pyM;
  long long I_M;
  // input: mask mode: obstacle bytes [layer][j][i] logical (1 obstacle, 0 free)
  const uint8_t* mask;
  // output: map mode -> physical ring layout [layer][py][px]; mask mode -> logical [layer][j][i]
  float* out;
  // scratch: per cell the column distances (rows) to the nearest obstacle / free cell, (dO | dF << 8),
  // logical [layer][j][i]
  uint16_t* g;
};
cudaError_t launch_sdf(const SdfParams& p, cudaStream_t s);

// ---- NEXT-3: trilinear query (query.cu) ---------------------------------------------------------------
// field 0: risk from the state records (stride 4 floats); field 1: sdf layers (stride 1, representative
// bins when paired); out 4 x n (value, d/dx, d/dy, d/dtheta); *n_out += queries with a corner outside
cudaError_t launch_trilinear(const float* field, int stride_elems, int is_sdf, const QueryGeo& g, int n,
                             const double* xyt, float* out, int* n_out, cudaStream_t s);

// ---- NEXT-4: nearest-neighbour inpainting of unknown cells (inpaint.cu) ------------------------------
// h: the elevation ring (NaN = unknown); site: logical [ny][nx] int scratch (nearest known row of the
// column); view: output ring (same layout as h); ctr[0] = known cells (zeroed by the caller), ctr[1..4] =
// logical bounding box (i_min, i_max, j_min, j_max) of the view cells whose value changed
// segs: inpaint_seg_ints(nx, ny) ints of scratch (per-segment first / last known rows)
cudaError_t launch_inpaint(const float* h, int ldh, int nx, int ny, int pxM, int pyM, int* site, float* view,
                           int* ctr, int* segs, cudaStream_t s);
size_t inpaint_seg_ints(int nx, int ny);

}  // namespace se2m
