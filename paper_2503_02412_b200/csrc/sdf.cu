// sdf.cu — NEXT-2: signed distance field of the explicit-obstacle set (Risk = 1) per yaw
// layer ("the corresponding signed distance field (SDF) will be generated"
// "the distance to the edge of the nearest region, with negative values inside obstacles"); reading R24:
// centre-to-centre Euclidean distance to the nearest cell of the other class, clamped to +-d_max.
//
// Exact within d_max by the separable Euclidean distance transform, in two kernels over whole layers:
//   sdf_cols_kernel  one thread per (column, 128-row segment): a downward and an upward sweep over the
//                    segment plus W = ceil(d_max / r) rows on each side give, per cell, the row distance
//                    to the nearest obstacle and to the nearest free cell of its column (255 beyond W);
//                    the class bit of a column is one word load + shift per row (consecutive threads =
//                    consecutive columns: the words are shared); the downward sweep is kept in shared
//                    memory, so each cell's (dO | dF << 8) is written to HBM once;
//   sdf_rows_kernel  one thread per cell: min over |dx| <= W of dx^2 + g(x + dx)^2 with g the column
//                    distance to the other class (squares staged in shared memory, "none" = a large
//                    sentinel, so the loop is branch-free; four offsets per step), stopping once dx^2
//                    reaches the best; a
//                    row-prefix count of the columns that have such a cell within W rejects cells with
//                    none in O(1).
#include <math.h>
#include <stdint.h>

#include "se2m_internal.h"

namespace se2m {

constexpr int SDF_SEG = 128;    // rows per column-pass thread
constexpr int SDF_ROWT = 256;   // columns per row-pass CTA

__global__ void __launch_bounds__(128) sdf_cols_kernel(const SdfParams p) {
  __shared__ uint16_t down[SDF_SEG][128];  // the downward sweep's (dO | dF << 8) of the segment's rows
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int L = blockIdx.z;
  if (i >= p.nx) return;
  const int j0 = blockIdx.y * SDF_SEG, j1 = min(p.ny, j0 + SDF_SEG);
  const int W = p.W;
  // class source of column i: map mode = one bit of a traversable word per row (physical rows, ring
  // order: the pointer wraps at ny); mask mode = one byte per row
  const uint32_t* tw = nullptr;
  int bit = 0;
  size_t tstride = 0;
  if (p.trav) {
    const long long I = p.I_M + i;
    const long long gI = I >= 0 ? I / 32 : -((-I + 31) / 32);
    const int wpos = (int)(((gI % p.trav_words) + p.trav_words) % p.trav_words);
    bit = (int)(I - gI * 32);
    tw = p.trav + (size_t)L * p.ny * p.trav_words + wpos;
    tstride = p.trav_words;
  }
  const uint8_t* mk = p.mask ? p.mask + (size_t)L * p.ny * p.nx + i : nullptr;
  auto obstacle = [&](int j, int py) -> int {
    return tw ? (int)(((__ldg(tw + py * tstride) >> bit) & 1u) ^ 1u) : (__ldg(mk + (size_t)j * p.nx) ? 1 : 0);
  };
  uint16_t* g = p.g + (size_t)L * p.ny * p.nx + i;  // (dO | dF << 8) per cell, logical [j][i]
  // downward: rows since the last obstacle / free cell, from W rows above the segment
  int dO = 255, dF = 255;
  int j = max(0, j0 - W);
  int py = p.pyM + j; if (py >= p.ny) py -= p.ny;
  for (; j < j1; ++j) {
    const int ob = obstacle(j, py);
    dO = ob ? 0 : min(dO + 1, 255);
    dF = ob ? min(dF + 1, 255) : 0;
    if (j >= j0) down[j - j0][threadIdx.x] = (uint16_t)(dO | (dF << 8));
    if (++py == p.ny) py = 0;
  }
  // upward, from W rows below the segment; keep the nearer one, clamp beyond W
  dO = dF = 255;
  j = min(p.ny, j1 + W) - 1;
  py = p.pyM + j; if (py >= p.ny) py -= p.ny;
  for (; j >= j0; --j) {
    const int ob = obstacle(j, py);
    dO = ob ? 0 : min(dO + 1, 255);
    dF = ob ? min(dF + 1, 255) : 0;
    if (j < j1) {
      const uint16_t v = down[j - j0][threadIdx.x];
      int o = min(dO, (int)(v & 0xff)), f = min(dF, (int)(v >> 8));
      if (o > W) o = 255;
      if (f > W) f = 255;
      g[(size_t)j * p.nx] = (uint16_t)(o | (f << 8));
    }
    if (--py < 0) py = p.ny - 1;
  }
}

__global__ void __launch_bounds__(SDF_ROWT) sdf_rows_kernel(const SdfParams p) {
  extern __shared__ unsigned char sm[];
  // the region reaches P = W + 3 columns past the tile on either side, so the scan below can test four
  // offsets per step; a candidate at |dx| > W lies beyond d_max (W = ceil(d_max / r)) and clamps to
  // d_max exactly like "none"
  const int W = p.W, P = W + 3, RW = SDF_ROWT + 2 * P;
  int* g2O = reinterpret_cast<int*>(sm);          // [RW] dO^2 (kFar: none within W / outside)
  int* g2F = g2O + RW;                            // [RW] dF^2
  unsigned short* cO = reinterpret_cast<unsigned short*>(g2F + RW);  // [RW + 1] prefix counts of dO <= W
  unsigned short* cF = cO + RW + 1;                                  // ... of dF <= W
  constexpr int kFar = 1 << 24;
  const int L = blockIdx.z, j = blockIdx.y, x0 = blockIdx.x * SDF_ROWT - P;
  const uint16_t* grow = p.g + ((size_t)L * p.ny + j) * p.nx;
  for (int c = threadIdx.x; c < RW; c += SDF_ROWT) {
    const int x = x0 + c;
    const uint16_t v = (x >= 0 && x < p.nx) ? grow[x] : (uint16_t)0xffff;  // outside the window: no cell
    const int o = v & 0xff, f = v >> 8;
    g2O[c] = o != 255 ? o * o : kFar;
    g2F[c] = f != 255 ? f * f : kFar;
  }
  __syncthreads();
  if (threadIdx.x < 64) {  // two warps: inclusive prefix counts along the region row (sequential chunks)
    const int lane = threadIdx.x & 31, which = threadIdx.x >> 5;
    unsigned short* cnt = which ? cF : cO;
    const int* g2 = which ? g2F : g2O;
    const int chunk = (RW + 31) / 32, c0 = min(RW, lane * chunk), c1 = min(RW, c0 + chunk);
    int run = 0;
    for (int c = c0; c < c1; ++c) run += g2[c] != kFar;
    int incl = run;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int acc = incl - run;
    if (lane == 0) cnt[0] = 0;
    for (int c = c0; c < c1; ++c) {
      acc += g2[c] != kFar;
      cnt[c + 1] = (unsigned short)acc;
    }
  }
  __syncthreads();
  const int x = x0 + P + threadIdx.x;
  if (x >= p.nx) return;
  const int c = P + threadIdx.x;
  const bool obst = g2O[c] == 0;          // own row distance to an obstacle is 0: the cell is one
  const int* g2 = obst ? g2F : g2O;       // distance to the other class
  const unsigned short* cnt = obst ? cF : cO;
  int best = kFar;
  if (cnt[c + W + 1] != cnt[c - W]) {     // some column within W has a cell of the other class
    best = g2[c];
    for (int dx = 1, dx2 = 1; dx <= W && dx2 < best; dx2 += 8 * dx + 16, dx += 4) {  // offsets dx .. dx + 3
      const int m0 = min(g2[c - dx], g2[c + dx]), m1 = min(g2[c - dx - 1], g2[c + dx + 1]);
      const int m2 = min(g2[c - dx - 2], g2[c + dx + 2]), m3 = min(g2[c - dx - 3], g2[c + dx + 3]);
      best = min(min(best, dx2 + m0), dx2 + 2 * dx + 1 + m1);
      best = min(min(best, dx2 + 4 * dx + 4 + m2), dx2 + 6 * dx + 9 + m3);
    }
  }
  float d = best >= kFar ? p.d_max : fminf(p.d_max, sqrtf((float)best) * p.r);
  if (obst) d = -d;
  size_t o;
  if (p.trav) {
    int px = p.pxM + x; if (px >= p.nx) px -= p.nx;
    int py = p.pyM + j; if (py >= p.ny) py -= p.ny;
    o = ((size_t)L * p.ny + py) * p.nx + px;
  } else {
    o = ((size_t)L * p.ny + j) * p.nx + x;
  }
  p.out[o] = d;
}

cudaError_t launch_sdf(const SdfParams& p, cudaStream_t s) {
  if (p.layers <= 0 || p.nx <= 0 || p.ny <= 0) return cudaSuccess;
  sdf_cols_kernel<<<dim3((p.nx + 127) / 128, (p.ny + SDF_SEG - 1) / SDF_SEG, p.layers), 128, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int RW = SDF_ROWT + 2 * (p.W + 3);
  const size_t smem = (size_t)RW * 8 + 2 * (size_t)(RW + 1) * 2;
  sdf_rows_kernel<<<dim3((p.nx + SDF_ROWT - 1) / SDF_ROWT, p.ny, p.layers), SDF_ROWT, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace se2m
