// se2m_internal.h — shared between the C-ABI runtime (se2map.cu) and the kernels (assess.cu).
// Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace se2m {

// Spatial tile of states handled by one CTA: world-aligned, TX = one warp.
constexpr int TX = 32;
constexpr int TY = 16;
constexpr int NTHREADS = 256;              // 8 warps; warp w owns tile rows w and w + 8
constexpr int ROWS_PER_WARP = TY / (NTHREADS / 32);

// Stencil radii the assess kernel is instantiated for (R_T >= the footprint radius R).
constexpr int kRadii[] = {4, 8, 12, 16, 24, 32};

struct AssessParams {
  // window / ring buffer: world cell (I, J) lives at physical (I mod nx, J mod ny)
  int nx, ny;            // window == ring dims
  int ldh;               // heights row pitch in floats (multiple of 4: 16-B TMA stride)
  long long I_M, J_M;    // window origin, world cells (Eq. 4)
  const float* h;        // [ny][ldh] physical, NaN = unknown
  // outputs, physical layout [k][ny][nx]; trav bits [k][ny][trav_words]
  float* risk;
  float* pitch;
  float* roll;
  float* z;
  uint32_t* trav;
  int trav_words;
  // yaw: rep bins k in [0, H); bin k + H (if paired) is the same footprint, x_yaw negated
  int n_yaw, H, paired;
  int R;                 // true footprint radius (cells); kernel template R_T >= R
  const int2* runs;      // [H][2*R_T+1] per stencil row dj = -R_T..R_T: di run [a, b]; empty = (0, -1)
  const float4* geo;     // [H] full-stencil (N, Sxx, Sxy, Syy) in cell units (Sx = Sy = 0)
  const float2* cs;      // [H] (cos, sin) of theta_k, k < H (reading R3)
  float r;               // resolution (m)
  // risk (Alg. 1 lines 10-18), all float
  float kappa_max, phi_x_max, phi_y_max;
  float wk, wx, wy;      // w_r[0]/kappa_max, w_r[1]/phi_x_max, w_r[2]/phi_y_max
  // tiles: world tile (TI, TJ) covers I in [TI*TX, TI*TX+TX), J in [TJ*TY, TJ*TY+TY)
  long long TI0, TJ0;    // first world tile of the dense tile grid
  int tiles_x;           // tile columns of the dense grid
  const int* tile_list;  // if non-null: linear indices (ty*tiles_x + tx) of the tiles to run
  int k_begin, k_end;    // representative-bin range this launch covers
  int k_chunk;           // rep bins per CTA (grid.y = ceil((k_end-k_begin)/k_chunk))
  int use_tma;           // tensor map valid
};

// Launch the assess kernel (one CTA per (tile, yaw chunk)).  Returns cudaSuccess or the launch error.
cudaError_t launch_assess(const AssessParams& p, int R_T, int n_tiles, const CUtensorMap* tmap,
                          cudaStream_t stream);

// Small helpers (same file as the kernels).
cudaError_t launch_clear_rect(float* h, int ldh, int x0, int y0, int w, int hgt, int nx, int ny,
                              cudaStream_t s);
cudaError_t launch_scatter_rect(float* h, int ldh, int nx, int ny, int px0, int py0, int w, int hgt,
                                const float* src, long long ld, const uint8_t* known, cudaStream_t s);
cudaError_t launch_gather_logical(const AssessParams& p, int k_lo, int k_hi, float* risk,
                                  float* pitch, float* roll, float* z, uint8_t* trav, cudaStream_t s);
cudaError_t launch_query(const AssessParams& p, int n, const int4* idx /* (px, py, k, valid) */,
                         float* out /* 5 x n: risk, pitch, roll, z, trav */, cudaStream_t s);

}  // namespace se2m
