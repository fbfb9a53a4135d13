// frontend.cu — NEXT-1: the elevation-map front-end of PAPER.md §V.A on the ring buffer.
//
//   fe_points_kernel   one thread per LiDAR point: sensor -> body -> world, map-range and
//                      body-frame height-band filters, sigma^2 = J_S^T S_S J_S + J_R^T S_R J_R
//                      + J_B^T S_B J_B;
//   fe_raycast_kernel  one warp per used point: the cells its ray crosses (lanes over the columns of the
//                      ray's major axis, each candidate confirmed by an exact slab test) are reset to
//                      unknown when their height exceeds the ray's highest height over the cell + eps
//                      (P:103);
//   (CUB stable radix sort of (cell, point index))
//   fe_fuse_kernel     one thread per cell run: the cell's points in input order through the 1-D Kalman
//                      filter with the Mahalanobis gate / higher-wins rule (readings R29-R30).
// All arithmetic is IEEE FP64 through __d*_rn intrinsics (no contraction), in the order the readings
// of DESIGN.md R26-R30 state, and cells store float32 height / variance after every update, so the
// result is a fixed function of the inputs (bit-identical to an FP64 evaluation in the same order).
#include <cub/device/device_radix_sort.cuh>
#include <math.h>
#include <stdint.h>

#include "se2m_internal.h"

namespace se2m {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }
// (a0*b0 + a1*b1) + a2*b2, left to right
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
  return da(da(dm(a0, b0), dm(a1, b1)), dm(a2, b2));
}
__device__ __forceinline__ double quad3(const double* S, double v0, double v1, double v2) {  // v^T S v
  const double s0 = dot3(S[0], S[1], S[2], v0, v1, v2), s1 = dot3(S[3], S[4], S[5], v0, v1, v2),
               s2 = dot3(S[6], S[7], S[8], v0, v1, v2);
  return dot3(v0, v1, v2, s0, s1, s2);
}

__global__ void fe_points_kernel(const FrontendArgs a, int n, const float* __restrict__ pts, int* __restrict__ key,
                                 int* __restrict__ idx, double4* __restrict__ meas, int* __restrict__ counts) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double* RB = a.pose.R_B;
  const double* RBS = a.pose.R_BS;
  const double p0 = pts[3 * (size_t)t], p1 = pts[3 * (size_t)t + 1], p2 = pts[3 * (size_t)t + 2];
  // q = R_BS p_S + p_BS (point in B); w = R_B q + p_B (world)
  const double q0 = da(dot3(RBS[0], RBS[1], RBS[2], p0, p1, p2), a.pose.p_BS[0]);
  const double q1 = da(dot3(RBS[3], RBS[4], RBS[5], p0, p1, p2), a.pose.p_BS[1]);
  const double q2 = da(dot3(RBS[6], RBS[7], RBS[8], p0, p1, p2), a.pose.p_BS[2]);
  const double x = da(dot3(RB[0], RB[1], RB[2], q0, q1, q2), a.pose.p_B[0]);
  const double y = da(dot3(RB[3], RB[4], RB[5], q0, q1, q2), a.pose.p_B[1]);
  const double z = da(dot3(RB[6], RB[7], RB[8], q0, q1, q2), a.pose.p_B[2]);
  // J_S = (R_B R_BS)^T b3 (third row of R_B R_BS); J_R = q x (third row of R_B); J_B = -b3
  const double js0 = dot3(RB[6], RB[7], RB[8], RBS[0], RBS[3], RBS[6]);
  const double js1 = dot3(RB[6], RB[7], RB[8], RBS[1], RBS[4], RBS[7]);
  const double js2 = dot3(RB[6], RB[7], RB[8], RBS[2], RBS[5], RBS[8]);
  const double jr0 = ds(dm(q1, RB[8]), dm(q2, RB[7])), jr1 = ds(dm(q2, RB[6]), dm(q0, RB[8])),
               jr2 = ds(dm(q0, RB[7]), dm(q1, RB[6]));
  double s2 = da(da(quad3(a.pose.Sigma_S, js0, js1, js2), quad3(a.pose.Sigma_R, jr0, jr1, jr2)),
                 quad3(a.pose.Sigma_B, 0.0, 0.0, -1.0));
  s2 = fmax(s2, 0.0);
  const long long I = (long long)floor(dd(x, a.r)), J = (long long)floor(dd(y, a.r));
  const long long i = I - a.I_M, j = J - a.J_M;
  int k = a.key_none, st = 0;
  if (!(i >= 0 && i < a.nx && j >= 0 && j < a.ny)) st = 1;            // outside the map
  else if (!(q2 >= a.z_min && q2 <= a.z_max)) st = 2;                   // height band in B
  else if (!(s2 > 0.0)) st = 3;                                         // unusable variance
  else {
    int px = a.pxM + (int)i; if (px >= a.nx) px -= a.nx;
    int py = a.pyM + (int)j; if (py >= a.ny) py -= a.ny;
    k = py * a.ldh + px;
  }
  key[t] = k;
  idx[t] = t;
  meas[t] = make_double4(x, y, z, s2);
  // status counters aggregated per warp (four words shared by the whole grid)
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int m = __popc(__ballot_sync(act, st == c));
    if (lane == leader && m) atomicAdd(counts + c, m);
  }
}

// Slab method (reading R28): parameter interval (t0, t1) of s + t d, t in (0, 1), inside the open square.
__device__ __forceinline__ bool cell_interval(double sx, double sy, double dx, double dy, double x0, double x1,
                                              double y0, double y1, double& t0, double& t1) {
  t0 = 0.0; t1 = 1.0;
  const double S[2] = {sx, sy}, D[2] = {dx, dy}, LO[2] = {x0, y0}, HI[2] = {x1, y1};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (D[c] == 0.0) {
      if (!(LO[c] < S[c] && S[c] < HI[c])) return false;
      continue;
    }
    double aa = dd(ds(LO[c], S[c]), D[c]), bb = dd(ds(HI[c], S[c]), D[c]);
    if (aa > bb) { const double tmp = aa; aa = bb; bb = tmp; }
    t0 = fmax(t0, aa);
    t1 = fmin(t1, bb);
  }
  return t0 < t1;
}

// One warp per ray: the lanes take the columns (x-major rays) or rows (y-major rays) of the ray's span;
// in its column a lane tests the (padded) range of rows the segment can cross there with the exact slab
// test of the oracle (reading R28), so the cells tested are a superset of the cells crossed and every
// decision is the oracle's.  All rays read the pre-frame heights; a cell reset by another ray reads
// NaN (unknown) and is left as it is, so the outcome does not depend on the order.
__global__ void fe_raycast_kernel(const FrontendArgs a, int n, const int* __restrict__ key,
                                  const double4* __restrict__ meas, float* h, int* bbox, int* n_reset) {
  const int t = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (t >= n || key[t] == a.key_none) return;  // warp-uniform
  const double4 e = meas[t];
  const double sx = a.sx, sy = a.sy, sz = a.sz;
  const double dx = ds(e.x, sx), dy = ds(e.y, sy), dz = ds(e.z, sz);
  const long long Ie = (long long)floor(dd(e.x, a.r)), Je = (long long)floor(dd(e.y, a.r));
  const long long Is = (long long)floor(dd(sx, a.r)), Js = (long long)floor(dd(sy, a.r));
  const bool xmaj = llabs(Ie - Is) >= llabs(Je - Js);
  // major axis (u) spans [u0, u1] cells; along the minor axis (w) the crossed cells lie between the
  // segment's w at the column's two faces (clipped to the segment), padded by one cell for rounding
  const long long u0 = xmaj ? min(Is, Ie) : min(Js, Je), u1 = xmaj ? max(Is, Ie) : max(Js, Je);
  const double su = xmaj ? sx : sy, sw = xmaj ? sy : sx, du = xmaj ? dx : dy, dw = xmaj ? dy : dx;
  int resets = 0, bi0 = 0x7fffffff, bi1 = -1, bj0 = 0x7fffffff, bj1 = -1;
  for (long long U = u0 + lane; U <= u1; U += 32) {
    double tlo = 0.0, thi = 1.0;
    if (du != 0.0) {
      double ta = dd(ds((double)U * a.r, su), du), tb = dd(ds((double)(U + 1) * a.r, su), du);
      if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
      tlo = fmax(0.0, ta);
      thi = fmin(1.0, tb);
    }
    const double wa = da(sw, dm(tlo, dw)), wb = da(sw, dm(thi, dw));
    const long long W0 = (long long)floor(dd(fmin(wa, wb), a.r)) - 1, W1 = (long long)floor(dd(fmax(wa, wb), a.r)) + 1;
    for (long long Wc = W0; Wc <= W1; ++Wc) {
      const long long I = xmaj ? U : Wc, J = xmaj ? Wc : U;
      if (I == Ie && J == Je) continue;  // the point's own cell is measured, not cleared (R28)
      const long long i = I - a.I_M, j = J - a.J_M;
      if (!(i >= 0 && i < a.nx && j >= 0 && j < a.ny)) continue;
      double t0, t1;
      if (!cell_interval(sx, sy, dx, dy, (double)I * a.r, (double)(I + 1) * a.r, (double)J * a.r,
                         (double)(J + 1) * a.r, t0, t1))
        continue;
      int px = a.pxM + (int)i; if (px >= a.nx) px -= a.nx;
      int py = a.pyM + (int)j; if (py >= a.ny) py -= a.ny;
      float* cell = h + (size_t)py * a.ldh + px;
      const float hc = *cell;
      const double zr = fmax(da(sz, dm(t0, dz)), da(sz, dm(t1, dz)));  // highest ray height over the cell
      if (!isnan(hc) && (double)hc > da(zr, a.ray_eps)) {              // P:103, margin reading R28
        *cell = __int_as_float(0x7fc00000);
        ++resets;
        bi0 = min(bi0, (int)i); bi1 = max(bi1, (int)i);
        bj0 = min(bj0, (int)j); bj1 = max(bj1, (int)j);
      }
    }
  }
  // one set of atomics per ray (warp): reset count and touched box
  resets = __reduce_add_sync(0xffffffffu, resets);
  bi0 = __reduce_min_sync(0xffffffffu, bi0); bi1 = __reduce_max_sync(0xffffffffu, bi1);
  bj0 = __reduce_min_sync(0xffffffffu, bj0); bj1 = __reduce_max_sync(0xffffffffu, bj1);
  if (lane == 0 && resets) {
    atomicAdd(n_reset, resets);
    atomicMin(bbox + 0, bi0); atomicMax(bbox + 1, bi1);
    atomicMin(bbox + 2, bj0); atomicMax(bbox + 3, bj1);
  }
}

__global__ void fe_fuse_kernel(const FrontendArgs a, int n, const int* __restrict__ skey, const int* __restrict__ sidx,
                               const double4* __restrict__ meas, float* h, float* var, int* bbox) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = t < n ? skey[t] : a.key_none;
  // one thread per run of equal cells; the touched-cell box is reduced per warp (one atomic per bound
  // and warp instead of per cell: the four bound words are shared by the whole grid)
  const bool lead = t < n && k != a.key_none && !(t > 0 && skey[t - 1] == k);
  int i = 0x7fffffff, j = 0x7fffffff, i1 = -1, j1 = -1;
  if (lead) {
    float* hp = h + k;
    float* vp = var + k;
    float hc = *hp, vc = *vp;
    // the run's measurements are gathered 8 at a time (independent loads in flight together) and
    // then fused in input order
    constexpr int CH = 8;
    for (int u0 = t; u0 < n && skey[u0] == k; u0 += CH) {
      double4 ech[CH];
      int cnt = 0;
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int u = u0 + q;
        const bool in = u < n && skey[u] == k;
        if (in) { ech[q] = meas[sidx[u]]; cnt = q + 1; }
      }
#pragma unroll
      for (int q = 0; q < CH; ++q) {
      if (q >= cnt) break;
      const double4 e = ech[q];
      const double z = e.z, s2 = e.w;
      if (isnan(hc)) { hc = (float)z; vc = (float)s2; continue; }  // unknown: initialise
      const double hh = hc, sc = vc;
      const double diff = fabs(ds(z, hh)), den = da(sc, s2);
      // Mahalanobis gate d = diff / sqrt(den) <= gate (reading R29), decided without the sqrt / division
      // chain unless d is within 1e-12 of the gate (then the exact formula, as in the oracle)
      const double l2 = dm(diff, diff), r2 = dm(dm(a.gate, a.gate), den);
      bool pass;
      if (l2 < r2 * (1.0 - 1e-12)) pass = true;
      else if (l2 > r2 * (1.0 + 1e-12)) pass = false;
      else pass = dd(diff, __dsqrt_rn(den)) <= a.gate;
      if (pass) {                                                     // 1-D Kalman update
        hc = (float)dd(da(dm(s2, hh), dm(sc, z)), den);
        vc = (float)dd(dm(sc, s2), den);
      } else if (z > hh) {                                            // Mahalanobis gate: higher wins
        hc = (float)z; vc = (float)s2;
      }
      }
      if (cnt < CH) break;
    }
    *hp = hc;
    *vp = vc;
    const int px = k % a.ldh, py = k / a.ldh;
    i = px >= a.pxM ? px - a.pxM : px + a.nx - a.pxM;
    j = py >= a.pyM ? py - a.pyM : py + a.ny - a.pyM;
    i1 = i; j1 = j;
  }
  i = __reduce_min_sync(0xffffffffu, i); i1 = __reduce_max_sync(0xffffffffu, i1);
  j = __reduce_min_sync(0xffffffffu, j); j1 = __reduce_max_sync(0xffffffffu, j1);
  if ((threadIdx.x & 31) == 0 && i1 >= 0) {
    atomicMin(bbox + 0, i); atomicMax(bbox + 1, i1);
    atomicMin(bbox + 2, j); atomicMax(bbox + 3, j1);
  }
}

cudaError_t frontend_run(const FrontendArgs& a, int n, const float* pts, FrontendScratch& s, float* h, float* var,
                         cudaStream_t st) {
  cudaError_t e;
  if (n <= 0) return cudaSuccess;
  const int B = 256, G = (n + B - 1) / B;
  fe_points_kernel<<<G, B, 0, st>>>(a, n, pts, s.key, s.idx, s.meas, s.counts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  fe_raycast_kernel<<<(unsigned)(((size_t)n * 32 + B - 1) / B), B, 0, st>>>(a, n, s.key, s.meas, h, s.bbox,
                                                                           s.counts + 4);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  size_t need = 0;
  // stable sort by cell over the key bits that occur (ring indices): the points of a cell keep their
  // input order (reading R29)
  cub::DeviceRadixSort::SortPairs(nullptr, need, s.key, s.skey, s.idx, s.sidx, n, 0, a.key_bits, st);
  if (need > s.temp_bytes) return cudaErrorMemoryAllocation;  // caller sizes the scratch (frontend_temp_bytes)
  e = cub::DeviceRadixSort::SortPairs(s.temp, need, s.key, s.skey, s.idx, s.sidx, n, 0, a.key_bits, st);
  if (e != cudaSuccess) return e;
  fe_fuse_kernel<<<G, B, 0, st>>>(a, n, s.skey, s.sidx, s.meas, h, var, s.bbox);
  return cudaGetLastError();
}

size_t frontend_temp_bytes(int n) {
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, (const int*)nullptr, (int*)nullptr, (const int*)nullptr, (int*)nullptr,
                                  n, 0, 32);
  return need;
}

}  // namespace se2m
