// assess.cu — sm_100a kernels of the SE(2) traversability hot path.
//
// assess_kernel<R_T>: Algorithm 1 (§V.B) for every state of one world-aligned
// TX x TY spatial tile and a chunk of yaw bins.  One CTA per (tile, yaw chunk):
//   1. the tile + an R_T-cell footprint halo of the ring-buffered elevation map lands in shared
//      memory, by one TMA box (cp.async.bulk.tensor.2d) when the halo lies inside the window and
//      does not straddle the ring seam, by coalesced LDG otherwise;
//   2. per halo row, exclusive prefix sums of h^ = h - h_ref, h^2, x' h^ (and, for tiles with
//      unknown / out-of-window cells, of the indicator v, x' v, x'^2 v) are built with warp scans;
//   3. for each representative yaw bin k < n_yaw/2 (reading R5: the ellipse depends on theta mod
//      pi), every state's footprint moments (FindEllipticalPoints + the covariance sums of Alg. 1
//      lines 1-8) are sums over the <= 2R+1 stencil rows of prefix differences: O(rows) per
//      state instead of O(cells) — an exact re-association of the sums of Alg. 1 lines 2-8;
//   4. register epilogue: covariance, closed-form smallest eigenpair + one inverse-iteration
//      refinement (GetMinEigenVecWithCurv, line 9), kappa, Eqs. 2-3 frame, pitch/roll (lines
//      12-13), thresholds and weighted risk (lines 10-18), written for bin k AND bin k + n/2
//      (x_yaw negated: pitch/roll negated, everything else identical — pin Q3);
//   5. coalesced stores to SoA planes + ballot-packed traversable bits.
// No tensor cores: the path is not a dense contraction.
#include <math.h>
#include <stdint.h>

#include "se2m_internal.h"

namespace se2m {

// ------------------------------------------------------------------------------------------
// TMA / mbarrier helpers (inline PTX, sm_90+ / sm_100a)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// ------------------------------------------------------------------------------------------
// Warp inclusive scan (Kogge-Stone), fixed order => deterministic rounding.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float warp_incl_scan(float v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

struct StateOut {
  float risk, pitch, roll, z;
  int trav;
};

// ------------------------------------------------------------------------------------------
// Register epilogue: moments -> covariance -> smallest eigenpair -> kappa, z, pitch, roll, risk.
// Moments are in cell units for x, y (dx = di*r) and metres for h^ = h - href.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ StateOut epilogue(float N, float Sx, float Sy, float Sxx, float Sxy, float Syy,
                                             float S0, float S2, float SXH, float SYH, float href,
                                             float2 csk, const AssessParams& p, bool general) {
  StateOut o;
  o.risk = 1.f;
  o.pitch = o.roll = o.z = __int_as_float(0x7fc00000);
  o.trav = 0;
  if (N < 2.5f) return o;  // |P| < 3: unknown (reading R8)
  const float invN = 1.f / N;
  const float mx = Sx * invN, my = Sy * invN, mh = S0 * invN;
  if (general) {
    // collinear footprint cells (exact integer moments): degenerate covariance (reading R11)
    const double dN = N;
    const double a = dN * Sxx - (double)Sx * Sx, b = dN * Syy - (double)Sy * Sy, c = dN * Sxy - (double)Sx * Sy;
    if (!(a * b - c * c > 1e-9 * a * b)) return o;
  }
  const float r = p.r, r2 = r * r;
  // Cov of Alg. 1 line 8 (divisor N), metres
  const float C00 = r2 * fmaf(-mx, mx, Sxx * invN);
  const float C01 = r2 * fmaf(-mx, my, Sxy * invN);
  const float C11 = r2 * fmaf(-my, my, Syy * invN);
  const float C02 = r * fmaf(-mx, mh, SXH * invN);
  const float C12 = r * fmaf(-my, mh, SYH * invN);
  const float C22 = fmaf(-mh, mh, S2 * invN);
  // smallest eigenvalue: trigonometric closed form on B = (C - q I)/p
  const float tr = C00 + C11 + C22;
  const float q = tr * (1.f / 3.f);
  const float b00 = C00 - q, b11 = C11 - q, b22 = C22 - q;
  const float p2 = b00 * b00 + b11 * b11 + b22 * b22 + 2.f * (C01 * C01 + C02 * C02 + C12 * C12);
  if (!(p2 > 0.f)) return o;  // isotropic: no unique normal
  const float pp = sqrtf(p2 * (1.f / 6.f));
  const float ip = 1.f / pp;
  const float d00 = b00 * ip, d11 = b11 * ip, d22 = b22 * ip, e01 = C01 * ip, e02 = C02 * ip, e12 = C12 * ip;
  const float detB = d00 * (d11 * d22 - e12 * e12) - e01 * (e01 * d22 - e12 * e02) + e02 * (e01 * e12 - d11 * e02);
  const float hr = fminf(1.f, fmaxf(-1.f, 0.5f * detB));
  const float phi = acosf(hr) * (1.f / 3.f);
  const float lam0 = fmaf(2.f * pp, cosf(phi + 2.09439510239319549f), q);
  // eigenvector: largest cross product of two rows of M = C - lam0 I (columns of adj(M))
  const float m00 = C00 - lam0, m11 = C11 - lam0, m22 = C22 - lam0;
  const float a0 = C01 * C12 - C02 * m11, a1 = C02 * C01 - m00 * C12, a2 = m00 * m11 - C01 * C01;  // r0 x r1
  const float b0 = C01 * m22 - C02 * C12, b1 = C02 * C02 - m00 * m22, b2 = m00 * C12 - C01 * C02;  // r0 x r2
  const float c0 = m11 * m22 - C12 * C12, c1 = C12 * C02 - C01 * m22, c2 = C01 * C12 - m11 * C02;  // r1 x r2
  const float na = a0 * a0 + a1 * a1 + a2 * a2, nb = b0 * b0 + b1 * b1 + b2 * b2, nc = c0 * c0 + c1 * c1 + c2 * c2;
  float v0, v1, v2;
  if (na >= nb && na >= nc) { v0 = a0; v1 = a1; v2 = a2; }
  else if (nb >= nc) { v0 = b0; v1 = b1; v2 = b2; }
  else { v0 = c0; v1 = c1; v2 = c2; }
  // one inverse-iteration step with the same shift: x = adj(M) v = v0 (r1 x r2) + v1 (r2 x r0) + v2 (r0 x r1)
  float x0 = v0 * c0 - v1 * b0 + v2 * a0;
  float x1 = v0 * c1 - v1 * b1 + v2 * a1;
  float x2 = v0 * c2 - v1 * b2 + v2 * a2;
  float nx2 = x0 * x0 + x1 * x1 + x2 * x2;
  if (!(nx2 > 0.f) || !isfinite(nx2)) {
    x0 = v0; x1 = v1; x2 = v2;
    nx2 = x0 * x0 + x1 * x1 + x2 * x2;
    if (!(nx2 > 0.f)) return o;
  }
  float inv = rsqrtf(nx2);
  if (x2 < 0.f) inv = -inv;  // z_b in S^2_+ 
  const float n0 = x0 * inv, n1 = x1 * inv, n2 = x2 * inv;
  if (!(n2 > 0.f)) return o;  // vertical plane: no S^2_+ normal (reading R11)
  // kappa_ter = lambda_min / trace (reading R1), lambda_min by the Rayleigh quotient of n
  const float t0 = C00 * n0 + C01 * n1 + C02 * n2;
  const float t1 = C01 * n0 + C11 * n1 + C12 * n2;
  const float t2 = C02 * n0 + C12 * n1 + C22 * n2;
  const float lmin = fmaxf(0.f, n0 * t0 + n1 * t1 + n2 * t2);
  const float kappa = lmin / tr;
  // z = f_1: fitted plane at the state centre (reading R14)
  o.z = href + mh + r * (n0 * mx + n1 * my) / n2;
  // Eqs. 2-3 reduced by the vector triple product: b3.x_b = -n_z u / |n x x_yaw|,
  // b3.y_b = (n_x sin - n_y cos) / |n x x_yaw|, |n x x_yaw|^2 = n_z^2 + (n_x sin - n_y cos)^2
  const float u = n0 * csk.x + n1 * csk.y;
  const float t = n0 * csk.y - n1 * csk.x;
  const float rs = rsqrtf(fmaf(n2, n2, t * t));
  const float sp = fminf(1.f, fmaxf(-1.f, -n2 * u * rs));
  const float sr = fminf(1.f, fmaxf(-1.f, t * rs));
  o.pitch = asinf(sp);
  o.roll = asinf(sr);
  const float ax = fabsf(o.pitch), ay = fabsf(o.roll);
  // Alg. 1 lines 10-18 (strict >, reading R15); risk = w . [k/kmax, phx/phxmax, phy/phymax]
  const bool early = (kappa > p.kappa_max) || (ax > p.phi_x_max) || (ay > p.phi_y_max);
  o.risk = early ? 1.f : fmaf(p.wk, kappa, fmaf(p.wx, ax, p.wy * ay));
  o.trav = early ? 0 : 1;
  return o;
}

// ------------------------------------------------------------------------------------------
// The assess kernel.
// ------------------------------------------------------------------------------------------
template <int R_T>
struct Geom {
  static constexpr int HX = TX + 2 * R_T;   // halo width (cells)
  static constexpr int HY = TY + 2 * R_T;   // halo height
  static constexpr int PW = HX + 1;         // prefix row length (exclusive prefix, entry 0 = 0)
  static constexpr int NR = 2 * R_T + 1;    // stencil rows
  static constexpr int CPL = (HX + 31) / 32;  // halo cells per lane in the row scan
  static constexpr size_t raw_bytes = ((size_t)HX * HY * 4 + 127) / 128 * 128;
  static constexpr size_t p02_off = raw_bytes;
  static constexpr size_t px_off = p02_off + (size_t)HY * PW * 8;
  static constexpr size_t pv_off = px_off + (size_t)HY * PW * 4;
  static constexpr size_t pvxx_off = pv_off + (size_t)HY * PW * 8;
  static constexpr size_t misc_off = (pvxx_off + (size_t)HY * PW * 4 + 15) / 16 * 16;
  // misc: mbarrier (8 B) + reduction scratch (3 x 8 words) + runs (k_chunk * NR int2)
  static constexpr size_t runs_off = misc_off + 128;
  static size_t bytes(int k_chunk) { return runs_off + (size_t)k_chunk * NR * 8; }
};

template <int R_T>
__global__ void __launch_bounds__(NTHREADS, 2)
    assess_kernel(const AssessParams p, const __grid_constant__ CUtensorMap tmap) {
  using G = Geom<R_T>;
  constexpr int HX = G::HX, HY = G::HY, PW = G::PW, NR = G::NR, CPL = G::CPL;
  extern __shared__ __align__(128) unsigned char smem[];
  float* raw = reinterpret_cast<float*>(smem);
  float2* p02 = reinterpret_cast<float2*>(smem + G::p02_off);
  float* pxh = reinterpret_cast<float*>(smem + G::px_off);
  float2* pv = reinterpret_cast<float2*>(smem + G::pv_off);
  float* pvxx = reinterpret_cast<float*>(smem + G::pvxx_off);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::misc_off);
  float* red = reinterpret_cast<float*>(smem + G::misc_off + 16);  // [3][8]
  int2* runs_s = reinterpret_cast<int2*>(smem + G::runs_off);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tlin = p.tile_list ? p.tile_list[blockIdx.x] : (int)blockIdx.x;
  const long long TI = p.TI0 + tlin % p.tiles_x;
  const long long TJ = p.TJ0 + tlin / p.tiles_x;
  const long long li0 = TI * TX - R_T - p.I_M;  // logical (window) index of halo column 0
  const long long lj0 = TJ * TY - R_T - p.J_M;
  const int kb = p.k_begin + blockIdx.y * p.k_chunk;
  const int ke = min(kb + p.k_chunk, p.k_end);
  if (kb >= ke) return;
  const int pxM = (int)(((p.I_M % p.nx) + p.nx) % p.nx);  // physical column of logical 0
  const int pyM = (int)(((p.J_M % p.ny) + p.ny) % p.ny);

  // ---- 1. halo -> shared memory ----------------------------------------------------------
  const bool box_in = li0 >= 0 && li0 + HX <= p.nx && lj0 >= 0 && lj0 + HY <= p.ny;
  int bx = 0, by = 0;
  if (box_in) {
    bx = pxM + (int)li0; if (bx >= p.nx) bx -= p.nx;
    by = pyM + (int)lj0; if (by >= p.ny) by -= p.ny;
  }
  const bool via_tma = p.use_tma && box_in && bx + HX <= p.nx && by + HY <= p.ny;
  if (via_tma) {
    if (tid == 0) {
      mbar_init(bar, 1);
      mbar_expect_tx(bar, (uint32_t)(HX * HY * 4));
      tma_load_2d(raw, &tmap, bar, bx, by);
    }
  } else {
    for (int idx = tid; idx < HX * HY; idx += NTHREADS) {
      const int row = idx / HX, col = idx - row * HX;
      const long long li = li0 + col, lj = lj0 + row;
      float v = __int_as_float(0x7fc00000);
      if (li >= 0 && li < p.nx && lj >= 0 && lj < p.ny) {
        int px = pxM + (int)li; if (px >= p.nx) px -= p.nx;
        int py = pyM + (int)lj; if (py >= p.ny) py -= p.ny;
        v = __ldg(p.h + (size_t)py * p.ldh + px);
      }
      raw[idx] = v;
    }
  }
  for (int idx = tid; idx < (ke - kb) * NR; idx += NTHREADS) runs_s[idx] = p.runs[(size_t)kb * NR + idx];
  __syncthreads();
  if (via_tma) mbar_wait(bar, 0);

  // ---- 2. validity + reference height (exact min/max: order-independent) --------------------
  float mn = INFINITY, mxv = -INFINITY;
  int allv = 1;
  for (int idx = tid; idx < HX * HY; idx += NTHREADS) {
    const float v = raw[idx];
    if (isnan(v)) allv = 0;
    else { mn = fminf(mn, v); mxv = fmaxf(mxv, v); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mxv = fmaxf(mxv, __shfl_xor_sync(0xffffffffu, mxv, o));
  }
  allv = __all_sync(0xffffffffu, allv);
  if (lane == 0) { red[warp] = mn; red[8 + warp] = mxv; red[16 + warp] = allv ? 1.f : 0.f; }
  __syncthreads();
  mn = red[0]; mxv = red[8];
  float allvf = red[16];
#pragma unroll
  for (int w = 1; w < NTHREADS / 32; ++w) { mn = fminf(mn, red[w]); mxv = fmaxf(mxv, red[8 + w]); allvf = fminf(allvf, red[16 + w]); }
  const bool fast = allvf > 0.5f;
  const float href = (mn <= mxv) ? 0.5f * (mn + mxv) : 0.f;

  // ---- 3. per-row exclusive prefix sums (warp w: rows w, w+8, ...) ---------------------------
  constexpr float XC = (float)(R_T + TX / 2);  // x' = col - XC; the state at lane l has x' = l - TX/2
  for (int row = warp; row < HY; row += NTHREADS / 32) {
    float e[CPL], e2[CPL], ex[CPL], vv[CPL], vx[CPL], vxx[CPL];
    float s0 = 0.f, s2 = 0.f, sx = 0.f, sv = 0.f, svx = 0.f, svxx = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int col = lane * CPL + c;
      float hv = (col < HX) ? raw[row * HX + col] : __int_as_float(0x7fc00000);
      const bool ok = !isnan(hv);
      const float hh = ok ? hv - href : 0.f;
      const float xp = (float)col - XC;
      s0 += hh; s2 = fmaf(hh, hh, s2); sx = fmaf(xp, hh, sx);
      e[c] = s0; e2[c] = s2; ex[c] = sx;
      if (!fast) {
        const float v = ok ? 1.f : 0.f;
        sv += v; svx = fmaf(xp, v, svx); svxx = fmaf(xp * xp, v, svxx);
        vv[c] = sv; vx[c] = svx; vxx[c] = svxx;
      }
    }
    // lane totals -> exclusive lane offsets
    const float o0 = warp_incl_scan(s0, lane) - s0;
    const float o2 = warp_incl_scan(s2, lane) - s2;
    const float ox = warp_incl_scan(sx, lane) - sx;
    float2* P02r = p02 + row * PW;
    float* PXr = pxh + row * PW;
    if (lane == 0) { P02r[0] = make_float2(0.f, 0.f); PXr[0] = 0.f; }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int col = lane * CPL + c;
      if (col < HX) { P02r[col + 1] = make_float2(o0 + e[c], o2 + e2[c]); PXr[col + 1] = ox + ex[c]; }
    }
    if (!fast) {
      const float ov = warp_incl_scan(sv, lane) - sv;
      const float ovx = warp_incl_scan(svx, lane) - svx;
      const float ovxx = warp_incl_scan(svxx, lane) - svxx;
      float2* PVr = pv + row * PW;
      float* PVXXr = pvxx + row * PW;
      if (lane == 0) { PVr[0] = make_float2(0.f, 0.f); PVXXr[0] = 0.f; }
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = lane * CPL + c;
        if (col < HX) { PVr[col + 1] = make_float2(ov + vv[c], ovx + vx[c]); PVXXr[col + 1] = ovxx + vxx[c]; }
      }
    }
  }
  __syncthreads();

  // ---- 4./5. states ------------------------------------------------------------------------
  const size_t plane = (size_t)p.nx * p.ny;
  const float xs = (float)(lane - TX / 2);
  const long long Iw = TI * TX + lane;
  const long long li = Iw - p.I_M;
  const bool col_in = li >= 0 && li < p.nx;
  int pxs = 0;
  if (col_in) { pxs = pxM + (int)li; if (pxs >= p.nx) pxs -= p.nx; }
  int rowv[ROWS_PER_WARP], pys[ROWS_PER_WARP];
  bool in[ROWS_PER_WARP];
#pragma unroll
  for (int s = 0; s < ROWS_PER_WARP; ++s) {
    rowv[s] = warp + s * (NTHREADS / 32);  // tile row
    const long long lj = TJ * TY + rowv[s] - p.J_M;
    in[s] = col_in && lj >= 0 && lj < p.ny;
    int py = 0;
    if (lj >= 0 && lj < p.ny) { py = pyM + (int)lj; if (py >= p.ny) py -= p.ny; }
    pys[s] = py;
  }
  const bool aligned_words = (p.nx % 32) == 0;

  for (int k = kb; k < ke; ++k) {
    const int2* rk = runs_s + (k - kb) * NR;
    const float4 g = __ldg(p.geo + k);
    const float2 csk = __ldg(p.cs + k);
    float S0[ROWS_PER_WARP], S2[ROWS_PER_WARP], SXH[ROWS_PER_WARP], SYH[ROWS_PER_WARP];
    float N[ROWS_PER_WARP], Sx[ROWS_PER_WARP], Sy[ROWS_PER_WARP], Sxx[ROWS_PER_WARP], Sxy[ROWS_PER_WARP],
        Syy[ROWS_PER_WARP];
#pragma unroll
    for (int s = 0; s < ROWS_PER_WARP; ++s) {
      S0[s] = S2[s] = SXH[s] = SYH[s] = 0.f;
      N[s] = Sx[s] = Sy[s] = Sxx[s] = Sxy[s] = Syy[s] = 0.f;
    }
    if (fast) {
#pragma unroll
      for (int d = 0; d < NR; ++d) {
        const int2 ab = rk[d];
        const float dj = (float)(d - R_T);
        const int c0 = lane + R_T + ab.x, c1 = lane + R_T + ab.y + 1;
#pragma unroll
        for (int s = 0; s < ROWS_PER_WARP; ++s) {
          const int row = rowv[s] + d;  // halo row of stencil row dj = d - R_T
          const float2 A = p02[row * PW + c0], B = p02[row * PW + c1];
          const float ax = pxh[row * PW + c0], bxv = pxh[row * PW + c1];
          const float d0 = B.x - A.x, d2 = B.y - A.y, dx = bxv - ax;
          S0[s] += d0;
          S2[s] += d2;
          SXH[s] += fmaf(-xs, d0, dx);
          SYH[s] = fmaf(dj, d0, SYH[s]);
        }
      }
#pragma unroll
      for (int s = 0; s < ROWS_PER_WARP; ++s) { N[s] = g.x; Sxx[s] = g.y; Sxy[s] = g.z; Syy[s] = g.w; }
    } else {
#pragma unroll
      for (int d = 0; d < NR; ++d) {
        const int2 ab = rk[d];
        const float dj = (float)(d - R_T);
        const int c0 = lane + R_T + ab.x, c1 = lane + R_T + ab.y + 1;
#pragma unroll
        for (int s = 0; s < ROWS_PER_WARP; ++s) {
          const int row = rowv[s] + d;
          const float2 A = p02[row * PW + c0], B = p02[row * PW + c1];
          const float ax = pxh[row * PW + c0], bxv = pxh[row * PW + c1];
          const float2 VA = pv[row * PW + c0], VB = pv[row * PW + c1];
          const float wa = pvxx[row * PW + c0], wb = pvxx[row * PW + c1];
          const float d0 = B.x - A.x, d2 = B.y - A.y, dx = bxv - ax;
          const float cnt = VB.x - VA.x, sxv = VB.y - VA.y, sxxv = wb - wa;  // exact integers
          const float sdi = fmaf(-xs, cnt, sxv);                              // sum di over the run
          S0[s] += d0;
          S2[s] += d2;
          SXH[s] += fmaf(-xs, d0, dx);
          SYH[s] = fmaf(dj, d0, SYH[s]);
          N[s] += cnt;
          Sx[s] += sdi;
          Sxx[s] += fmaf(xs * xs, cnt, fmaf(-2.f * xs, sxv, sxxv));
          Sy[s] = fmaf(dj, cnt, Sy[s]);
          Syy[s] = fmaf(dj * dj, cnt, Syy[s]);
          Sxy[s] = fmaf(dj, sdi, Sxy[s]);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < ROWS_PER_WARP; ++s) {
      const StateOut o = epilogue(N[s], Sx[s], Sy[s], Sxx[s], Sxy[s], Syy[s], S0[s], S2[s], SXH[s], SYH[s], href,
                                  csk, p, !fast);
      const size_t off = (size_t)pys[s] * p.nx + pxs;
      if (in[s]) {
        p.risk[(size_t)k * plane + off] = o.risk;
        p.pitch[(size_t)k * plane + off] = o.pitch;
        p.roll[(size_t)k * plane + off] = o.roll;
        p.z[(size_t)k * plane + off] = o.z;
        if (p.paired) {
          const size_t k2 = (size_t)(k + p.H);
          p.risk[k2 * plane + off] = o.risk;
          p.pitch[k2 * plane + off] = -o.pitch;
          p.roll[k2 * plane + off] = -o.roll;
          p.z[k2 * plane + off] = o.z;
        }
      }
      const unsigned inmask = __ballot_sync(0xffffffffu, in[s]);
      const unsigned tmask = __ballot_sync(0xffffffffu, in[s] && o.trav);
      if (inmask == 0xffffffffu && aligned_words) {
        if (lane == 0) {
          const size_t w = ((size_t)k * p.ny + pys[s]) * p.trav_words + (pxs >> 5);
          p.trav[w] = tmask;
          if (p.paired) p.trav[((size_t)(k + p.H) * p.ny + pys[s]) * p.trav_words + (pxs >> 5)] = tmask;
        }
      } else if (in[s]) {
        const unsigned bit = 1u << (pxs & 31);
        const size_t w = ((size_t)k * p.ny + pys[s]) * p.trav_words + (pxs >> 5);
        if (o.trav) atomicOr(p.trav + w, bit); else atomicAnd(p.trav + w, ~bit);
        if (p.paired) {
          const size_t w2 = ((size_t)(k + p.H) * p.ny + pys[s]) * p.trav_words + (pxs >> 5);
          if (o.trav) atomicOr(p.trav + w2, bit); else atomicAnd(p.trav + w2, ~bit);
        }
      }
    }
  }
}

template <int R_T>
static cudaError_t launch_t(const AssessParams& p, int n_tiles, const CUtensorMap* tmap, cudaStream_t stream) {
  using G = Geom<R_T>;
  const size_t smem = G::bytes(p.k_chunk);
  static int configured_bytes = 0;
  if ((int)smem > configured_bytes) {
    cudaError_t e = cudaFuncSetAttribute(assess_kernel<R_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured_bytes = (int)smem;
  }
  const int nk = p.k_end - p.k_begin;
  dim3 grid(n_tiles, (nk + p.k_chunk - 1) / p.k_chunk);
  assess_kernel<R_T><<<grid, NTHREADS, smem, stream>>>(p, *tmap);
  return cudaGetLastError();
}

cudaError_t launch_assess(const AssessParams& p, int R_T, int n_tiles, const CUtensorMap* tmap, cudaStream_t stream) {
  if (n_tiles <= 0 || p.k_end <= p.k_begin) return cudaSuccess;
  switch (R_T) {
    case 4: return launch_t<4>(p, n_tiles, tmap, stream);
    case 8: return launch_t<8>(p, n_tiles, tmap, stream);
    case 12: return launch_t<12>(p, n_tiles, tmap, stream);
    case 16: return launch_t<16>(p, n_tiles, tmap, stream);
    case 24: return launch_t<24>(p, n_tiles, tmap, stream);
    case 32: return launch_t<32>(p, n_tiles, tmap, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------
// Ring-buffer helpers: clear (H1), scatter (H2), logical gather (download), query (H10).
// ------------------------------------------------------------------------------------------
__global__ void clear_rect_kernel(float* h, int ldh, int x0, int y0, int w, int hgt, int nx, int ny) {
  // (x0, y0): physical start; the rectangle wraps modulo (nx, ny)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= w || j >= hgt) return;
  int px = x0 + i; if (px >= nx) px -= nx;
  int py = y0 + j; if (py >= ny) py -= ny;
  h[(size_t)py * ldh + px] = __int_as_float(0x7fc00000);
}

cudaError_t launch_clear_rect(float* h, int ldh, int x0, int y0, int w, int hgt, int nx, int ny, cudaStream_t s) {
  if (w <= 0 || hgt <= 0) return cudaSuccess;
  dim3 grid((w + 255) / 256, hgt);
  clear_rect_kernel<<<grid, 256, 0, s>>>(h, ldh, x0, y0, w, hgt, nx, ny);
  return cudaGetLastError();
}

__global__ void scatter_rect_kernel(float* h, int ldh, int nx, int ny, int px0, int py0, int w, int hgt,
                                    const float* __restrict__ src, long long ld, const uint8_t* __restrict__ known) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= w || j >= hgt) return;
  int px = px0 + i; if (px >= nx) px -= nx;
  int py = py0 + j; if (py >= ny) py -= ny;
  const size_t si = (size_t)j * ld + i;
  float v = src[si];
  if (known && !known[si]) v = __int_as_float(0x7fc00000);
  h[(size_t)py * ldh + px] = v;
}

cudaError_t launch_scatter_rect(float* h, int ldh, int nx, int ny, int px0, int py0, int w, int hgt, const float* src,
                                long long ld, const uint8_t* known, cudaStream_t s) {
  if (w <= 0 || hgt <= 0) return cudaSuccess;
  dim3 grid((w + 255) / 256, hgt);
  scatter_rect_kernel<<<grid, 256, 0, s>>>(h, ldh, nx, ny, px0, py0, w, hgt, src, ld, known);
  return cudaGetLastError();
}

__global__ void gather_logical_kernel(const AssessParams p, int k_lo, int k_hi, int pxM, int pyM, float* risk,
                                      float* pitch, float* roll, float* z, uint8_t* trav) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i >= p.nx) return;
  int px = pxM + i; if (px >= p.nx) px -= p.nx;
  int py = pyM + j; if (py >= p.ny) py -= p.ny;
  const size_t src = ((size_t)k * p.ny + py) * p.nx + px;
  const size_t dst = ((size_t)k * p.ny + j) * p.nx + i;
  const bool owned = k >= k_lo && k < k_hi;
  const float qnan = __int_as_float(0x7fc00000);
  if (risk) risk[dst] = owned ? p.risk[src] : qnan;
  if (pitch) pitch[dst] = owned ? p.pitch[src] : qnan;
  if (roll) roll[dst] = owned ? p.roll[src] : qnan;
  if (z) z[dst] = owned ? p.z[src] : qnan;
  if (trav) trav[dst] = owned ? (uint8_t)((p.trav[((size_t)k * p.ny + py) * p.trav_words + (px >> 5)] >> (px & 31)) & 1u) : 0;
}

cudaError_t launch_gather_logical(const AssessParams& p, int k_lo, int k_hi, float* risk, float* pitch, float* roll,
                                  float* z, uint8_t* trav, cudaStream_t s) {
  const int pxM = (int)(((p.I_M % p.nx) + p.nx) % p.nx);
  const int pyM = (int)(((p.J_M % p.ny) + p.ny) % p.ny);
  dim3 grid((p.nx + 255) / 256, p.ny, p.n_yaw);
  gather_logical_kernel<<<grid, 256, 0, s>>>(p, k_lo, k_hi, pxM, pyM, risk, pitch, roll, z, trav);
  return cudaGetLastError();
}

__global__ void query_kernel(const AssessParams p, int n, const int4* __restrict__ idx, float* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int4 e = idx[q];
  const float qnan = __int_as_float(0x7fc00000);
  float r = qnan, pi = qnan, ro = qnan, zz = qnan, tv = 0.f;
  if (e.w) {
    const size_t o = ((size_t)e.z * p.ny + e.y) * p.nx + e.x;
    r = p.risk[o]; pi = p.pitch[o]; ro = p.roll[o]; zz = p.z[o];
    tv = (float)((p.trav[((size_t)e.z * p.ny + e.y) * p.trav_words + (e.x >> 5)] >> (e.x & 31)) & 1u);
  }
  out[q] = r; out[n + q] = pi; out[2 * (size_t)n + q] = ro; out[3 * (size_t)n + q] = zz; out[4 * (size_t)n + q] = tv;
}

cudaError_t launch_query(const AssessParams& p, int n, const int4* idx, float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  query_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, n, idx, out);
  return cudaGetLastError();
}

}  // namespace se2m
