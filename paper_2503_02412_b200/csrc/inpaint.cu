// inpaint.cu — NEXT-4: nearest-neighbour inpainting of the window ("can be inpainted by
// classical methods"; "nearest-neighbor interpolation for elevation inpainting").
// Reading R31: every unknown cell takes the height of its nearest known cell of the window,
// Euclidean distance on (logical) grid indices, ties to the known cell first in row-major (j, i) order.
//
// Exact separable search (integer arithmetic only, heights are copied):
//   inpaint_seg/cols     per logical column: for every cell the nearest known row of its column (ties: the
//                        upper one = row-major first within a column), by 32-row segments;
//   inpaint_rows_kernel  one thread per cell: columns x' = i, i +- 1, ... outward, candidate distance
//                        (i - x')^2 + (j - site(x'))^2, lexicographic (distance, site row, x') minimum; the
//                        search stops once (i - x')^2 exceeds the best distance.  Any column's nearest
//                        known cell is its vertically nearest one, and within a column the upper of two
//                        equidistant cells precedes the lower in row-major order, so the minimum over
//                        the per-column candidates is the row-major-first nearest known cell.
#include <cuda_runtime.h>
#include <stdint.h>

#include "se2m_internal.h"

namespace se2m {

// Column pass in two kernels over (column, 32-row segment) threads — consecutive threads are
// consecutive columns, so every access is coalesced, and nx * ny / 32 threads keep the GPU busy even
// on tall windows: segment summaries (first / last known row), then each thread resolves its segment
// with the nearest known rows above / below it found among the other segments' summaries.
constexpr int kSeg = 32;

__global__ void inpaint_seg_kernel(const float* __restrict__ h, int ldh, int nx, int ny, int pxM, int pyM,
                                   int* __restrict__ first, int* __restrict__ last, int* __restrict__ ctr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = blockIdx.y;
  if (blockIdx.x == 0 && seg == 0 && threadIdx.x == 0) {  // changed-cell box, used by the rows pass
    ctr[1] = nx; ctr[2] = -1; ctr[3] = ny; ctr[4] = -1;
  }
  int known = 0;
  if (i < nx) {
    int px = pxM + i;
    if (px >= nx) px -= nx;
    const int j0 = seg * kSeg, j1 = min(ny, j0 + kSeg);
    int py = pyM + j0;
    if (py >= ny) py -= ny;
    int f = -1, l = -1;
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {
      if (!isnan(h[(size_t)py * ldh + px])) { if (f < 0) f = j; l = j; ++known; }
      if (++py == ny) py = 0;
    }
    first[(size_t)seg * nx + i] = f;
    last[(size_t)seg * nx + i] = l;
  }
  // block-reduce the known count into one atomic
  for (int o = 16; o > 0; o >>= 1) known += __shfl_xor_sync(0xffffffffu, known, o);
  if ((threadIdx.x & 31) == 0 && known) atomicAdd(ctr, known);
}

__global__ void inpaint_cols_kernel(const float* __restrict__ h, int ldh, int nx, int ny, int pxM, int pyM,
                                    const int* __restrict__ first, const int* __restrict__ last,
                                    int* __restrict__ site) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = blockIdx.y, nseg = gridDim.y;
  if (i >= nx) return;
  int up = -1, dn = -1;  // nearest known row above the segment / below it
  for (int s = seg - 1; s >= 0 && up < 0; --s) up = last[(size_t)s * nx + i];
  for (int s = seg + 1; s < nseg && dn < 0; ++s) dn = first[(size_t)s * nx + i];
  int px = pxM + i;
  if (px >= nx) px -= nx;
  const int j0 = seg * kSeg, j1 = min(ny, j0 + kSeg);
  int py = pyM + j0;
  if (py >= ny) py -= ny;
  int* col = site + i;
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {  // downward: nearest known row at or above j
    if (!isnan(h[(size_t)py * ldh + px])) up = j;
    col[(size_t)j * nx] = up;
    if (++py == ny) py = 0;
  }
  py = pyM + j1 - 1;
  if (py >= ny) py -= ny;
#pragma unroll 4
  for (int j = j1 - 1; j >= j0; --j) {  // upward: nearest known row at or below j; ties stay with the upper
    if (!isnan(h[(size_t)py * ldh + px])) dn = j;
    const int a = col[(size_t)j * nx];
    col[(size_t)j * nx] = (a < 0 || (dn >= 0 && dn - j < j - a)) ? dn : a;
    if (--py < 0) py = ny - 1;
  }
}

__global__ void inpaint_rows_kernel(const float* __restrict__ h, int ldh, int nx, int ny, int pxM, int pyM,
                                    const int* __restrict__ site, float* __restrict__ view, int* __restrict__ ctr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= nx) return;
  const int* srow = site + (size_t)j * nx;
  long long best = 0x7fffffffffffffffLL;
  int bs = -1, bx = -1;
  for (int d = 0;; ++d) {
    const long long dd = (long long)d * d;
    if (dd > best || (i - d < 0 && i + d >= nx)) break;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      if (side == 1 && d == 0) break;
      const int x = side ? i + d : i - d;
      if (x < 0 || x >= nx) continue;
      const int s = __ldg(srow + x);
      if (s < 0) continue;
      const long long D = dd + (long long)(j - s) * (j - s);
      if (D < best || (D == best && (s < bs || (s == bs && x < bx)))) { best = D; bs = s; bx = x; }
    }
  }
  int px = pxM + i, py = pyM + j;
  if (px >= nx) px -= nx;
  if (py >= ny) py -= ny;
  float v = __int_as_float(0x7fc00000);  // no known cell anywhere: stays unknown
  if (bs >= 0) {
    int sx = pxM + bx, sy = pyM + bs;
    if (sx >= nx) sx -= nx;
    if (sy >= ny) sy -= ny;
    v = h[(size_t)sy * ldh + sx];
  }
  float* dst = view + (size_t)py * ldh + px;
  if (__float_as_uint(*dst) != __float_as_uint(v)) {
    *dst = v;
    atomicMin(ctr + 1, i); atomicMax(ctr + 2, i); atomicMin(ctr + 3, j); atomicMax(ctr + 4, j);
  }
}

cudaError_t launch_inpaint(const float* h, int ldh, int nx, int ny, int pxM, int pyM, int* site, float* view,
                           int* ctr, int* segs, cudaStream_t s) {
  const int nseg = (ny + kSeg - 1) / kSeg;
  int* first = segs;
  int* last = segs + (size_t)nseg * nx;
  inpaint_seg_kernel<<<dim3((nx + 127) / 128, nseg), 128, 0, s>>>(h, ldh, nx, ny, pxM, pyM, first, last, ctr);
  inpaint_cols_kernel<<<dim3((nx + 127) / 128, nseg), 128, 0, s>>>(h, ldh, nx, ny, pxM, pyM, first, last, site);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  inpaint_rows_kernel<<<dim3((nx + 255) / 256, ny), 256, 0, s>>>(h, ldh, nx, ny, pxM, pyM, site, view, ctr);
  return cudaGetLastError();
}

size_t inpaint_seg_ints(int nx, int ny) { return 2 * (size_t)((ny + kSeg - 1) / kSeg) * nx; }

}  // namespace se2m
