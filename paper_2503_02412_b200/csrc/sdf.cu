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
//                    memory (so each cell's (dO | dF << 8) is written to HBM once, and the upward sweep
//                    reads the segment's class bits back from it: dO = 0 <=> obstacle);
//   sdf_rows_kernel  4 or 8 cells per thread, 1024 or 2048 columns of one row per CTA: min over
//                    |dx| <= W of dx^2 + g(x + dx)^2 with g the column distance to the other class
//                    (squares staged in shared memory, "none" = a large sentinel, so the loop is
//                    branch-free; four offsets per step), stopping once dx^2 reaches the best; one flag
//                    bit per column and class (warp ballots while staging: the column has a cell of the
//                    class within W rows) rejects cells with none within W columns by testing the <= 2W + 1
//                    bits of their window, word by word.
#include <math.h>
#include <stdint.h>

#include "se2m_internal.h"

namespace se2m {

#ifndef SE2M_SDF_SEG
#define SE2M_SDF_SEG 128
#endif
#ifndef SE2M_SDF_PAIRS
#define SE2M_SDF_PAIRS 1  // row pass over pairs of neighbouring cells (sdf_rows_pair_kernel)
#endif
constexpr int SDF_SEG = SE2M_SDF_SEG;  // rows per column-pass thread
constexpr int SDF_ROWT = 256;          // threads per row-pass CTA
// cells per row-pass thread (a CTA: SDF_ROWT * CPT columns of one row): 8 on rows wider than 1536 columns, else 4
// (one CTA per row segment amortises the staging; A/B in profiles/r02_ab.md)

template <bool MAP>  // class source: MAP = the map's traversable bits, else an obstacle-byte mask
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
  if (MAP) {
    const long long I = p.I_M + i;
    const long long gI = I >= 0 ? I / 32 : -((-I + 31) / 32);
    const int wpos = (int)(((gI % p.trav_words) + p.trav_words) % p.trav_words);
    bit = (int)(I - gI * 32);
    tw = p.trav + (size_t)L * p.ny * p.trav_words + wpos;
    tstride = p.trav_words;
  }
  const uint8_t* mk = MAP ? nullptr : p.mask + (size_t)L * p.ny * p.nx + i;
  auto obstacle = [&](int j, int py) -> int {
    if (MAP) return (int)(((__ldg(tw + py * tstride) >> bit) & 1u) ^ 1u);
    return __ldg(mk + (size_t)j * p.nx) ? 1 : 0;
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
  // upward, from W rows below the segment (their class bits from memory); keep the nearer one, clamp beyond W
  dO = dF = 255;
  j = min(p.ny, j1 + W) - 1;
  py = p.pyM + j; if (py >= p.ny) py -= p.ny;
  for (; j >= j1; --j) {
    const int ob = obstacle(j, py);
    dO = ob ? 0 : min(dO + 1, 255);
    dF = ob ? min(dF + 1, 255) : 0;
    if (--py < 0) py = p.ny - 1;
  }
  for (j = j1 - 1; j >= j0; --j) {  // the segment: its class bits from the downward sweep (dO = 0 <=> obstacle)
    const uint16_t v = down[j - j0][threadIdx.x];
    const int ob = (v & 0xff) == 0;
    dO = ob ? 0 : min(dO + 1, 255);
    dF = ob ? min(dF + 1, 255) : 0;
    int o = min(dO, (int)(v & 0xff)), f = min(dF, (int)(v >> 8));
    if (o > W) o = 255;
    if (f > W) f = 255;
    g[(size_t)j * p.nx] = (uint16_t)(o | (f << 8));
  }
}

template <int SDF_CPT>
__global__ void __launch_bounds__(SDF_ROWT) sdf_rows_kernel(const SdfParams p) {
  extern __shared__ unsigned char sm[];
  // the region reaches P = W + 3 columns past the CTA's span on either side, so the scan below can test four
  // offsets per step; a candidate at |dx| > W lies beyond d_max (W = ceil(d_max / r)) and clamps to d_max
  // exactly like "none"
  constexpr int SPAN = SDF_ROWT * SDF_CPT;
  const int W = p.W, P = W + 3, RW = SPAN + 2 * P, NWD = (RW + 31) / 32 + 1;  // (+1: the two-word window read)
  int* g2O = reinterpret_cast<int*>(sm);          // [RW] dO^2 (kFar: none within W / outside)
  int* g2F = g2O + RW;                            // [RW] dF^2
  unsigned* bO = reinterpret_cast<unsigned*>(g2F + RW);  // [NWD] bit c: column c has an obstacle within W rows
  if (threadIdx.x < 2) bO[threadIdx.x * NWD + NWD - 1] = 0u;  // the spare word of each class
  unsigned* bF = bO + NWD;                               // ... a free cell within W rows
  constexpr int kFar = 1 << 24;
  const int L = blockIdx.z, j = blockIdx.y, x0 = blockIdx.x * SPAN - P;
  const int lane = threadIdx.x & 31;
  const uint16_t* grow = p.g + ((size_t)L * p.ny + j) * p.nx;
  // a warp stages 32 consecutive region columns per step (warp-uniform loop): one ballot per class = one word
  for (int c0 = threadIdx.x & ~31; c0 < RW; c0 += SDF_ROWT) {
    const int c = c0 + lane, x = x0 + c;
    const uint16_t v = (c < RW && x >= 0 && x < p.nx) ? grow[x] : (uint16_t)0xffff;  // outside the window: no cell
    const int o = v & 0xff, f = v >> 8;
    if (c < RW) {
      g2O[c] = o != 255 ? o * o : kFar;
      g2F[c] = f != 255 ? f * f : kFar;
    }
    const unsigned wo = __ballot_sync(0xffffffffu, o != 255), wf = __ballot_sync(0xffffffffu, f != 255);
    if (lane == 0) { bO[c0 >> 5] = wo; bF[c0 >> 5] = wf; }
  }
  __syncthreads();
#pragma unroll 1
  for (int i = 0; i < SDF_CPT; ++i) {
    const int c = P + threadIdx.x + i * SDF_ROWT;
    const int x = x0 + c;
    if (x0 + P + i * SDF_ROWT >= p.nx) break;  // (warp-uniform: the whole CTA's step i is past the row)
    const bool valid = x < p.nx;             // (region columns past the row hold "none": reads stay in bounds)
    const bool obst = g2O[c] == 0;          // own row distance to an obstacle is 0: the cell is one
    const int* g2 = obst ? g2F : g2O;       // distance to the other class
    const unsigned* bw = obst ? bF : bO;
    // some column in [c - W, c + W] has a cell of the other class within W rows?
    const int a = c - W, b = c + W, wa = a >> 5, wb = b >> 5;
    unsigned long long any;
    if (W <= 31) {  // the 2W + 1 window bits lie in words wa, wa + 1
      const unsigned long long w64 = ((unsigned long long)bw[wa + 1] << 32) | bw[wa];
      any = (w64 >> (a & 31)) & ((2ull << (2 * W)) - 1ull);
    } else {
      any = 0;
#pragma unroll 1
      for (int w = wa; w <= wb; ++w) {
        unsigned m = bw[w];
        if (w == wa) m &= 0xffffffffu << (a & 31);
        if (w == wb) m &= 0xffffffffu >> (31 - (b & 31));
        any |= m;
      }
    }
    const bool scan = valid && any != 0ull;
    int best = scan ? g2[c] : kFar;
    // offsets dx .. dx + 3 per step, the step warp-uniform (dx and its squares are the same in every lane) until
    // no lane of the warp can improve: a lane whose dx^2 reached its best only takes mins that cannot lower it
    const int* pl = g2 + (c - 1);
    const int* pr = g2 + (c + 1);
    int s0 = 1, t = 3;  // dx^2 and 2 dx + 1 of the step's first offset
#pragma unroll 1
    for (int dx = 1; dx <= W; dx += 4, pl -= 4, pr += 4) {
      if (!__any_sync(0xffffffffu, scan && s0 < best)) break;
      const int s1 = s0 + t, s2 = s1 + t + 2, s3 = s2 + t + 4;  // (dx + 1)^2, (dx + 2)^2, (dx + 3)^2
      best = min(best, s0 + min(pl[0], pr[0]));
      best = min(best, s1 + min(pl[-1], pr[1]));
      best = min(best, s2 + min(pl[-2], pr[2]));
      best = min(best, s3 + min(pl[-3], pr[3]));
      s0 = s3 + t + 6;  // (dx + 4)^2
      t += 8;
    }
    if (!valid) continue;
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
}

// Row pass over PAIRS of neighbouring cells (x, x + 1): when both are of one class they scan one set of candidate
// columns — a candidate d columns left of x is d + 1 left of x + 1, one right of x + 1 is one further from x — so
// each candidate load serves both cells; a pair of mixed classes is two cells at distance 1 from the other class.
// Same results as sdf_rows_kernel (candidates past W clamp to d_max either way).
template <int PPT>
__global__ void __launch_bounds__(SDF_ROWT) sdf_rows_pair_kernel(const SdfParams p) {
  extern __shared__ unsigned char sm[];
  constexpr int SPAN = SDF_ROWT * 2 * PPT;
  const int W = p.W, P = W + 4, RW = SPAN + 2 * P, NWD = (RW + 31) / 32 + 1;
  int* g2O = reinterpret_cast<int*>(sm);
  int* g2F = g2O + RW;
  unsigned* bO = reinterpret_cast<unsigned*>(g2F + RW);
  if (threadIdx.x < 2) bO[threadIdx.x * NWD + NWD - 1] = 0u;
  unsigned* bF = bO + NWD;
  constexpr int kFar = 1 << 24;
  const int L = blockIdx.z, j = blockIdx.y, x0 = blockIdx.x * SPAN - P;
  const int lane = threadIdx.x & 31;
  const uint16_t* grow = p.g + ((size_t)L * p.ny + j) * p.nx;
  for (int c0 = threadIdx.x & ~31; c0 < RW; c0 += SDF_ROWT) {
    const int c = c0 + lane, x = x0 + c;
    const uint16_t v = (c < RW && x >= 0 && x < p.nx) ? grow[x] : (uint16_t)0xffff;
    const int o = v & 0xff, f = v >> 8;
    if (c < RW) {
      g2O[c] = o != 255 ? o * o : kFar;
      g2F[c] = f != 255 ? f * f : kFar;
    }
    const unsigned wo = __ballot_sync(0xffffffffu, o != 255), wf = __ballot_sync(0xffffffffu, f != 255);
    if (lane == 0) { bO[c0 >> 5] = wo; bF[c0 >> 5] = wf; }
  }
  __syncthreads();
  const int py = p.trav ? (p.pyM + j >= p.ny ? p.pyM + j - p.ny : p.pyM + j) : 0;
#pragma unroll 1
  for (int i = 0; i < PPT; ++i) {
    const int c = P + 2 * (threadIdx.x + i * SDF_ROWT);  // the pair's left cell (region column)
    const int x = x0 + c;
    if (x0 + P + 2 * i * SDF_ROWT >= p.nx) break;  // (CTA-uniform)
    const bool va = x < p.nx, vb = x + 1 < p.nx;
    const bool oa = g2O[c] == 0, ob = g2O[c + 1] == 0;
    const bool mixed = vb && oa != ob;
    const int* g2 = oa ? g2F : g2O;
    const unsigned* bw = oa ? bF : bO;
    // some column in [c - W, c + 1 + W] has a cell of the other class within W rows?
    const int a = c - W, b = c + 1 + W, wa = a >> 5, wb = b >> 5;
    unsigned long long any;
    if (W <= 30) {  // the 2W + 2 window bits lie in words wa, wa + 1
      const unsigned long long w64 = ((unsigned long long)bw[wa + 1] << 32) | bw[wa];
      any = (w64 >> (a & 31)) & ((4ull << (2 * W)) - 1ull);
    } else {
      any = 0;
#pragma unroll 1
      for (int w = wa; w <= wb; ++w) {
        unsigned m = bw[w];
        if (w == wa) m &= 0xffffffffu << (a & 31);
        if (w == wb) m &= 0xffffffffu >> (31 - (b & 31));
        any |= m;
      }
    }
    const bool scan = va && !mixed && any != 0ull;
    int ba = scan ? min(g2[c], 1 + g2[c + 1]) : kFar;
    int bb = scan ? min(g2[c + 1], 1 + g2[c]) : kFar;
    if (mixed) ba = bb = 1;
    const int* pl = g2 + (c - 1);  // candidates d .. d + 3 left of x
    const int* pr = g2 + (c + 2);  // ... right of x + 1
    int s0 = 1, t = 3;             // d^2, 2 d + 1
#pragma unroll 1
    for (int d = 1; d <= W; d += 4, pl -= 4, pr += 4) {
      if (!__any_sync(0xffffffffu, scan && s0 < max(ba, bb))) break;
      const int s1 = s0 + t, s2 = s1 + t + 2, s3 = s2 + t + 4, s4 = s3 + t + 6;  // (d + 1)^2 .. (d + 4)^2
      const int l0 = pl[0], l1 = pl[-1], l2 = pl[-2], l3 = pl[-3];
      const int r0 = pr[0], r1 = pr[1], r2 = pr[2], r3 = pr[3];
      ba = min(min(ba, s0 + l0), s1 + r0);
      bb = min(min(bb, s0 + r0), s1 + l0);
      ba = min(min(ba, s1 + l1), s2 + r1);
      bb = min(min(bb, s1 + r1), s2 + l1);
      ba = min(min(ba, s2 + l2), s3 + r2);
      bb = min(min(bb, s2 + r2), s3 + l2);
      ba = min(min(ba, s3 + l3), s4 + r3);
      bb = min(min(bb, s3 + r3), s4 + l3);
      s0 = s4;
      t += 8;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(h ? vb : va)) continue;
      const int best = h ? bb : ba;
      float d = best >= kFar ? p.d_max : fminf(p.d_max, sqrtf((float)best) * p.r);
      if (h ? ob : oa) d = -d;
      size_t o;
      if (p.trav) {
        int px = p.pxM + x + h; if (px >= p.nx) px -= p.nx;
        o = ((size_t)L * p.ny + py) * p.nx + px;
      } else {
        o = ((size_t)L * p.ny + j) * p.nx + x + h;
      }
      p.out[o] = d;
    }
  }
}

cudaError_t launch_sdf(const SdfParams& p, cudaStream_t s) {
  if (p.layers <= 0 || p.nx <= 0 || p.ny <= 0) return cudaSuccess;
  const dim3 gc((p.nx + 127) / 128, (p.ny + SDF_SEG - 1) / SDF_SEG, p.layers);
  if (p.trav) sdf_cols_kernel<true><<<gc, 128, 0, s>>>(p);
  else sdf_cols_kernel<false><<<gc, 128, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int cpt = p.nx > 1536 ? 8 : 4;
  const int SPAN = SDF_ROWT * cpt;
  if (SE2M_SDF_PAIRS) {
    const int RW = SPAN + 2 * (p.W + 4);
    const size_t smem = (size_t)RW * 8 + 2 * (size_t)((RW + 31) / 32 + 1) * 4;
    const dim3 gr((p.nx + SPAN - 1) / SPAN, p.ny, p.layers);
    if (cpt == 8) sdf_rows_pair_kernel<4><<<gr, SDF_ROWT, smem, s>>>(p);
    else sdf_rows_pair_kernel<2><<<gr, SDF_ROWT, smem, s>>>(p);
    return cudaGetLastError();
  }
  const int RW = SPAN + 2 * (p.W + 3);
  const size_t smem = (size_t)RW * 8 + 2 * (size_t)((RW + 31) / 32 + 1) * 4;
  const dim3 gr((p.nx + SPAN - 1) / SPAN, p.ny, p.layers);
  if (cpt == 8) sdf_rows_kernel<8><<<gr, SDF_ROWT, smem, s>>>(p);
  else sdf_rows_kernel<4><<<gr, SDF_ROWT, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace se2m
