// sdf.cu — NEXT-2: signed distance field of the explicit-obstacle set (Risk = 1) per yaw
// layer ("the corresponding signed distance field (SDF) will be generated"
// "the distance to the edge of the nearest region, with negative values inside obstacles"); reading R24:
// centre-to-centre Euclidean distance to the nearest cell of the other class, clamped to +-d_max.
//
// Exact within d_max: one CTA per 32 x 32 tile of one layer loads the class of every cell of the tile
// plus a W = ceil(d_max / r) halo into shared memory, computes per column the distance (in rows) to the
// nearest obstacle / free cell within W (separable first pass of an EDT), then per cell the minimum of
// dx^2 + g(x + dx)^2 over |dx| <= W with early exit once dx^2 exceeds the best (second pass).  The
// column distances come from per-column bit masks (ffs / clz), O(1) per entry.
#include <math.h>
#include <stdint.h>

#include "se2m_internal.h"

namespace se2m {

constexpr int SDF_T = 32;
constexpr int SDF_THREADS = 256;

__global__ void __launch_bounds__(SDF_THREADS) sdf_kernel(const SdfParams p) {
  extern __shared__ unsigned char sm[];
  const int W = p.W, RW = SDF_T + 2 * W;  // region width / height
  unsigned char* cls = sm;                 // [RW][RW]: 0 free, 1 obstacle, 2 outside the window
  unsigned char* gO = cls + RW * RW;       // [SDF_T][RW]: rows to the nearest obstacle in the column (255 none)
  unsigned char* gF = gO + SDF_T * RW;     // ... to the nearest free cell
  const int tiles_x = (p.nx + SDF_T - 1) / SDF_T;
  const int i0 = (blockIdx.x % tiles_x) * SDF_T, j0 = (blockIdx.x / tiles_x) * SDF_T;
  const int L = blockIdx.y;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < RW * RW; idx += SDF_THREADS) {
    const int rj = idx / RW, ri = idx - rj * RW;
    const int i = i0 - W + ri, j = j0 - W + rj;
    unsigned char c = 2;
    if (i >= 0 && i < p.nx && j >= 0 && j < p.ny) {
      if (p.trav) {
        int py = p.pyM + j; if (py >= p.ny) py -= p.ny;
        const long long I = p.I_M + i;
        const long long g = I >= 0 ? I / 32 : -((-I + 31) / 32);
        const int w = (int)(((g % p.trav_words) + p.trav_words) % p.trav_words);
        const uint32_t word = p.trav[((size_t)L * p.ny + py) * p.trav_words + w];
        c = ((word >> (int)(I - g * 32)) & 1u) ? 0 : 1;  // traversable -> free, Risk = 1 -> obstacle
      } else {
        c = p.mask[((size_t)L * p.ny + j) * p.nx + i] ? 1 : 0;
      }
    }
    cls[idx] = c;
  }
  __syncthreads();
  // pass 1: per region column a bit mask over the region's rows of obstacle / free cells (one thread per
  // column), then per (tile row, column) the distance to the nearest set bit by ffs / clz (O(1))
  uint64_t* mO = reinterpret_cast<uint64_t*>(((uintptr_t)(gF + SDF_T * RW) + 7) & ~(uintptr_t)7);
  const int NWd = (RW + 63) >> 6;          // 64-bit words per column mask (<= 4 for W <= 96)
  uint64_t* mF = mO + (size_t)RW * NWd;
  for (int c = tid; c < RW; c += SDF_THREADS) {
    for (int w = 0; w < NWd; ++w) {
      uint64_t o = 0, f = 0;
      for (int b = 0; b < 64; ++b) {
        const int rr = w * 64 + b;
        if (rr >= RW) break;
        const unsigned char v = cls[rr * RW + c];
        o |= (uint64_t)(v == 1) << b;
        f |= (uint64_t)(v == 0) << b;
      }
      mO[c * NWd + w] = o;
      mF[c * NWd + w] = f;
    }
  }
  __syncthreads();
  auto nearest = [&](const uint64_t* m, int r) {  // rows from row r to the nearest set bit, 255 beyond W
    const int w = r >> 6, b = r & 63;
    int up = 1 << 20, dn = 1 << 20;
    const uint64_t x = m[w] >> b;
    if (x) up = __ffsll((long long)x) - 1;
    else
      for (int w2 = w + 1; w2 < NWd; ++w2)
        if (m[w2]) { up = w2 * 64 + __ffsll((long long)m[w2]) - 1 - r; break; }
    const uint64_t y = m[w] << (63 - b);
    if (y) dn = __clzll((long long)y);
    else
      for (int w2 = w - 1; w2 >= 0; --w2)
        if (m[w2]) { dn = r - (w2 * 64 + 63 - __clzll((long long)m[w2])); break; }
    const int d = min(up, dn);
    return d <= W ? d : 255;
  };
  for (int idx = tid; idx < SDF_T * RW; idx += SDF_THREADS) {
    const int ty = idx / RW, c = idx - ty * RW;
    gO[ty * RW + c] = (unsigned char)nearest(mO + c * NWd, ty + W);
    gF[ty * RW + c] = (unsigned char)nearest(mF + c * NWd, ty + W);
  }
  __syncthreads();
  // pass 2: per tile cell, nearest cell of the other class
  for (int idx = tid; idx < SDF_T * SDF_T; idx += SDF_THREADS) {
    const int ty = idx / SDF_T, tx = idx - ty * SDF_T;
    const int i = i0 + tx, j = j0 + ty;
    if (i >= p.nx || j >= p.ny) continue;
    const int c = tx + W;
    const unsigned char self = cls[(ty + W) * RW + c];
    const unsigned char* g = (self == 1 ? gF : gO) + ty * RW;
    int best = 0x7fffffff;
    for (int dx = 0; dx <= W && dx * dx < best; ++dx) {
      const int a = g[c - dx], b = g[c + dx];
      if (a != 255) best = min(best, dx * dx + a * a);
      if (b != 255) best = min(best, dx * dx + b * b);
    }
    float d = best == 0x7fffffff ? p.d_max : fminf(p.d_max, sqrtf((float)best) * p.r);
    if (self == 1) d = -d;
    size_t o;
    if (p.trav) {
      int px = p.pxM + i; if (px >= p.nx) px -= p.nx;
      int py = p.pyM + j; if (py >= p.ny) py -= p.ny;
      o = ((size_t)L * p.ny + py) * p.nx + px;
    } else {
      o = ((size_t)L * p.ny + j) * p.nx + i;
    }
    p.out[o] = d;
  }
}

cudaError_t launch_sdf(const SdfParams& p, cudaStream_t s) {
  if (p.layers <= 0 || p.nx <= 0 || p.ny <= 0) return cudaSuccess;
  const int RW = SDF_T + 2 * p.W;
  const size_t smem = (size_t)RW * RW + 2 * (size_t)SDF_T * RW + 8 + 2 * (size_t)RW * ((RW + 63) / 64) * 8;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(sdf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int tiles = ((p.nx + SDF_T - 1) / SDF_T) * ((p.ny + SDF_T - 1) / SDF_T);
  sdf_kernel<<<dim3(tiles, p.layers), SDF_THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace se2m
