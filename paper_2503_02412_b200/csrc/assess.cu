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
//   5. coalesced 16-B stores of (risk, pitch, roll, z) state records + ballot-packed traversable bits.
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

// Packed FP32x2 (sm_100a FADD2): two lanes of arithmetic per issue slot.
__device__ __forceinline__ unsigned long long f2_bits(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 bits_f2(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}
// MUFU approximations (relative error ~1 ulp); the eigenvector refinement absorbs them.
__device__ __forceinline__ float frcp(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float fsqrt(float x) { float r; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
// acos on [-1, 1]: Abramowitz & Stegun 4.4.46, acos(a) = sqrt(1 - a) * P7(a) for a in [0, 1].
__device__ __forceinline__ float acos_fast(float x) {
  const float a = fabsf(x);
  float pz = fmaf(-0.0012624911f, a, 0.0066700901f);
  pz = fmaf(pz, a, -0.0170881256f);
  pz = fmaf(pz, a, 0.0308918810f);
  pz = fmaf(pz, a, -0.0501743046f);
  pz = fmaf(pz, a, 0.0889789874f);
  pz = fmaf(pz, a, -0.2145988016f);
  pz = fmaf(pz, a, 1.5707963050f);
  const float r = fsqrt(1.f - a) * pz;
  return x < 0.f ? 3.14159265358979f - r : r;
}
// asin on [-1, 1], branch-free Cephes asinf (odd: asin(-x) = -asin(x), asin(0) = 0 exactly).
__device__ __forceinline__ float asin_fast(float x) {
  const float a = fabsf(x);
  const bool big = a > 0.5f;
  const float z = big ? 0.5f * (1.f - a) : a * a;
  const float s = big ? fsqrt(z) : a;
  float pz = fmaf(4.2163199048e-2f, z, 2.4181311049e-2f);
  pz = fmaf(pz, z, 4.5470025998e-2f);
  pz = fmaf(pz, z, 7.4953002686e-2f);
  pz = fmaf(pz, z, 1.6666752422e-1f);
  float r = fmaf(s * z, pz, s);
  r = big ? fmaf(-2.f, r, 1.57079632679489662f) : r;
  return copysignf(r, x);
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
  const float invN = frcp(N);
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
  const float p2 = (b00 * b00 + b11 * b11 + b22 * b22 + 2.f * (C01 * C01 + C02 * C02 + C12 * C12)) * (1.f / 6.f);
  if (!(p2 > 0.f)) return o;  // isotropic: no unique normal
  const float ip = rsqrtf(p2);
  const float pp = p2 * ip;
  const float d00 = b00 * ip, d11 = b11 * ip, d22 = b22 * ip, e01 = C01 * ip, e02 = C02 * ip, e12 = C12 * ip;
  const float detB = d00 * (d11 * d22 - e12 * e12) - e01 * (e01 * d22 - e12 * e02) + e02 * (e01 * e12 - d11 * e02);
  const float hr = fminf(1.f, fmaxf(-1.f, 0.5f * detB));
  const float phi = acos_fast(hr) * (1.f / 3.f);
  float sphi, cphi;
  __sincosf(phi, &sphi, &cphi);
  const float lam0 = fmaf(-pp, fmaf(1.73205080756887729f, sphi, cphi), q);  // q + 2p cos(phi + 2pi/3)
  // eigenvector: largest cross product of two rows of M = C - lam0 I (columns of adj(M))
  const float m00 = C00 - lam0, m11 = C11 - lam0, m22 = C22 - lam0;
  const float a0 = C01 * C12 - C02 * m11, a1 = C02 * C01 - m00 * C12, a2 = m00 * m11 - C01 * C01;  // r0 x r1
  const float b0 = C01 * m22 - C02 * C12, b1 = C02 * C02 - m00 * m22, b2 = m00 * C12 - C01 * C02;  // r0 x r2
  const float c0 = m11 * m22 - C12 * C12, c1 = C12 * C02 - C01 * m22, c2 = C01 * C12 - m11 * C02;  // r1 x r2
  const float na = a0 * a0 + a1 * a1 + a2 * a2, nb = b0 * b0 + b1 * b1 + b2 * b2, nc = c0 * c0 + c1 * c1 + c2 * c2;
  const bool pa = na >= nb && na >= nc, pb = !pa && nb >= nc;
  const float v0 = pa ? a0 : (pb ? b0 : c0), v1 = pa ? a1 : (pb ? b1 : c1), v2 = pa ? a2 : (pb ? b2 : c2);
  // one inverse-iteration step with the same shift: x = adj(M) v = v0 (r1 x r2) + v1 (r2 x r0) + v2 (r0 x r1)
  float x0 = v0 * c0 - v1 * b0 + v2 * a0;
  float x1 = v0 * c1 - v1 * b1 + v2 * a1;
  float x2 = v0 * c2 - v1 * b2 + v2 * a2;
  float nx2 = x0 * x0 + x1 * x1 + x2 * x2;
  if (!(nx2 > 0.f) || !(nx2 < 3.0e38f)) {
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
  const float kappa = lmin * frcp(tr);
  // z = f_1: fitted plane at the state centre (reading R14)
  o.z = href + fmaf(r * (n0 * mx + n1 * my), frcp(n2), mh);
  // Eqs. 2-3 reduced by the vector triple product: b3.x_b = -n_z u / |n x x_yaw|,
  // b3.y_b = (n_x sin - n_y cos) / |n x x_yaw|, |n x x_yaw|^2 = n_z^2 + (n_x sin - n_y cos)^2
  const float u = n0 * csk.x + n1 * csk.y;
  const float t = n0 * csk.y - n1 * csk.x;
  const float rs = rsqrtf(fmaf(n2, n2, t * t));
  const float sp = fminf(1.f, fmaxf(-1.f, -n2 * u * rs));
  const float sr = fminf(1.f, fmaxf(-1.f, t * rs));
  o.pitch = asin_fast(sp);
  o.roll = asin_fast(sr);
  const float ax = fabsf(o.pitch), ay = fabsf(o.roll);
  // Alg. 1 lines 10-18 (strict >, reading R15); risk = w . [k/kmax, phx/phxmax, phy/phymax]
  const bool early = (kappa > p.kappa_max) || (ax > p.phi_x_max) || (ay > p.phi_y_max);
  o.risk = early ? 1.f : fmaf(p.wk, kappa, fmaf(p.wx, ax, p.wy * ay));
  o.trav = early ? 0 : 1;
  return o;
}

// ------------------------------------------------------------------------------------------
// Packed two-state epilogue for interior tiles (all footprint cells known and inside the window).
// Every FP32 add/mul/fma runs as one sm_100a FADD2/FMUL2/FFMA2 on (state a, state b); MUFU, compares
// and selects run per lane.  The footprint geometry is the per-bin constant gc = (C00, C01, C11, 1/N),
// gd = (r/N, C00 + C11, C01^2, -) (metres, computed in FP64 on the host), so Sx = Sy = 0, mx = my = 0.
// ------------------------------------------------------------------------------------------
struct F2 {
  unsigned long long v;
};
__device__ __forceinline__ F2 pk(float a, float b) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ F2 bc(float a) { return pk(a, a); }
__device__ __forceinline__ float lo(F2 x) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v)); return a; }
__device__ __forceinline__ float hi(F2 x) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v)); return b; }
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { F2 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v)); return d; }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { F2 d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v)); return d; }
__device__ __forceinline__ F2 operator*(F2 a, F2 b) { F2 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v)); return d; }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return d;
}
template <class Fn>
__device__ __forceinline__ F2 map2(F2 x, Fn f) { return pk(f(lo(x)), f(hi(x))); }

__device__ __forceinline__ F2 acos2(F2 x) {  // A&S 4.4.46, packed polynomial
  const float xl = lo(x), xh = hi(x);
  const F2 a = pk(fabsf(xl), fabsf(xh));
  F2 pz = fma2(bc(-0.0012624911f), a, bc(0.0066700901f));
  pz = fma2(pz, a, bc(-0.0170881256f));
  pz = fma2(pz, a, bc(0.0308918810f));
  pz = fma2(pz, a, bc(-0.0501743046f));
  pz = fma2(pz, a, bc(0.0889789874f));
  pz = fma2(pz, a, bc(-0.2145988016f));
  pz = fma2(pz, a, bc(1.5707963050f));
  const F2 om = bc(1.f) - a;
  const F2 r = pk(fsqrt(lo(om)), fsqrt(hi(om))) * pz;
  const float rl = lo(r), rh = hi(r);
  return pk(xl < 0.f ? 3.14159265358979f - rl : rl, xh < 0.f ? 3.14159265358979f - rh : rh);
}
__device__ __forceinline__ F2 asin2(F2 x) {  // Cephes asinf, packed polynomial; odd, asin(0) = 0
  const float xl = lo(x), xh = hi(x);
  const float al = fabsf(xl), ah = fabsf(xh);
  const bool bl = al > 0.5f, bh = ah > 0.5f;
  const F2 a = pk(al, ah);
  const F2 sq = a * a;
  const F2 half = fma2(bc(-0.5f), a, bc(0.5f));  // (1 - a) / 2
  const F2 z = pk(bl ? lo(half) : lo(sq), bh ? hi(half) : hi(sq));
  const F2 sv = pk(bl ? fsqrt(lo(z)) : al, bh ? fsqrt(hi(z)) : ah);
  F2 pz = fma2(bc(4.2163199048e-2f), z, bc(2.4181311049e-2f));
  pz = fma2(pz, z, bc(4.5470025998e-2f));
  pz = fma2(pz, z, bc(7.4953002686e-2f));
  pz = fma2(pz, z, bc(1.6666752422e-1f));
  const F2 r = fma2(sv * z, pz, sv);
  const F2 big = fma2(bc(-2.f), r, bc(1.57079632679489662f));
  return pk(copysignf(bl ? lo(big) : lo(r), xl), copysignf(bh ? hi(big) : hi(r), xh));
}

struct StateOut2 {
  F2 risk, pitch, roll, z;
  unsigned trav_a, trav_b;
};

__device__ __forceinline__ StateOut2 epilogue2(F2 S0, F2 S2, F2 SXH, F2 SYH, float href, float4 gc, float4 gd,
                                               float2 csk, const AssessParams& p) {
  const F2 mh = S0 * bc(gc.w);
  const F2 C02 = SXH * bc(gd.x), C12 = SYH * bc(gd.x);
  const F2 C22 = fma2(mh * bc(-1.f), mh, S2 * bc(gc.w));
  const F2 tr = C22 + bc(gd.y);
  const F2 q = tr * bc(1.f / 3.f);
  const F2 b00 = bc(gc.x) - q, b11 = bc(gc.z) - q, b22 = C22 - q;
  F2 p2 = fma2(C02, C02, fma2(C12, C12, bc(gd.z)));
  p2 = p2 + p2;
  p2 = fma2(b00, b00, fma2(b11, b11, fma2(b22, b22, p2)));
  p2 = p2 * bc(1.f / 6.f);
  const float p2l = lo(p2), p2h = hi(p2);
  const bool okl = p2l > 0.f, okh = p2h > 0.f;  // isotropic covariance: no unique normal
  const F2 ip = pk(rsqrtf(okl ? p2l : 1.f), rsqrtf(okh ? p2h : 1.f));
  const F2 pp = p2 * ip;
  const F2 d00 = b00 * ip, d11 = b11 * ip, d22 = b22 * ip, e01 = bc(gc.y) * ip, e02 = C02 * ip, e12 = C12 * ip;
  // det(B/p) = d00 (d11 d22 - e12^2) - e01 (e01 d22 - e12 e02) + e02 (e01 e12 - d11 e02)
  const F2 m1 = fma2(d11, d22, (e12 * e12) * bc(-1.f));
  const F2 m2 = fma2(e01, d22, (e12 * e02) * bc(-1.f));
  const F2 m3 = fma2(e01, e12, (d11 * e02) * bc(-1.f));
  const F2 detB = fma2(e02, m3, fma2(d00, m1, (e01 * m2) * bc(-1.f)));
  const F2 hr = pk(fminf(1.f, fmaxf(-1.f, 0.5f * lo(detB))), fminf(1.f, fmaxf(-1.f, 0.5f * hi(detB))));
  const F2 phi = acos2(hr) * bc(1.f / 3.f);
  float sl, cl, sh, ch;
  __sincosf(lo(phi), &sl, &cl);
  __sincosf(hi(phi), &sh, &ch);
  const F2 lam0 = fma2(pp * bc(-1.f), fma2(bc(1.73205080756887729f), pk(sl, sh), pk(cl, ch)), q);
  // eigenvector: largest cross product of two rows of M = C - lam0 I; one inverse-iteration step
  const F2 C00 = bc(gc.x), C01 = bc(gc.y), C11 = bc(gc.z);
  const F2 m00 = C00 - lam0, m11 = C11 - lam0, m22 = C22 - lam0;
  const F2 a0 = fma2(C01, C12, (C02 * m11) * bc(-1.f)), a1 = fma2(C02, C01, (m00 * C12) * bc(-1.f)),
           a2 = fma2(m00, m11, (C01 * C01) * bc(-1.f));
  const F2 b0 = fma2(C01, m22, (C02 * C12) * bc(-1.f)), b1 = fma2(C02, C02, (m00 * m22) * bc(-1.f)),
           b2 = fma2(m00, C12, (C01 * C02) * bc(-1.f));
  const F2 c0 = fma2(m11, m22, (C12 * C12) * bc(-1.f)), c1 = fma2(C12, C02, (C01 * m22) * bc(-1.f)),
           c2 = fma2(C01, C12, (m11 * C02) * bc(-1.f));
  const F2 na = fma2(a0, a0, fma2(a1, a1, a2 * a2)), nb = fma2(b0, b0, fma2(b1, b1, b2 * b2)),
           nc = fma2(c0, c0, fma2(c1, c1, c2 * c2));
  const bool pal = lo(na) >= lo(nb) && lo(na) >= lo(nc), pbl = !pal && lo(nb) >= lo(nc);
  const bool pah = hi(na) >= hi(nb) && hi(na) >= hi(nc), pbh = !pah && hi(nb) >= hi(nc);
  const F2 v0 = pk(pal ? lo(a0) : (pbl ? lo(b0) : lo(c0)), pah ? hi(a0) : (pbh ? hi(b0) : hi(c0)));
  const F2 v1 = pk(pal ? lo(a1) : (pbl ? lo(b1) : lo(c1)), pah ? hi(a1) : (pbh ? hi(b1) : hi(c1)));
  const F2 v2 = pk(pal ? lo(a2) : (pbl ? lo(b2) : lo(c2)), pah ? hi(a2) : (pbh ? hi(b2) : hi(c2)));
  const F2 x0 = fma2(v0, c0, fma2(v1 * bc(-1.f), b0, v2 * a0));
  const F2 x1 = fma2(v0, c1, fma2(v1 * bc(-1.f), b1, v2 * a1));
  const F2 x2 = fma2(v0, c2, fma2(v1 * bc(-1.f), b2, v2 * a2));
  const F2 nx2 = fma2(x0, x0, fma2(x1, x1, x2 * x2));
  const F2 nv2 = fma2(v0, v0, fma2(v1, v1, v2 * v2));
  // fall back to the unrefined vector if the refinement under/overflowed
  const bool rl = lo(nx2) > 0.f && lo(nx2) < 3.0e38f, rh = hi(nx2) > 0.f && hi(nx2) < 3.0e38f;
  const F2 y0 = pk(rl ? lo(x0) : lo(v0), rh ? hi(x0) : hi(v0));
  const F2 y1 = pk(rl ? lo(x1) : lo(v1), rh ? hi(x1) : hi(v1));
  const F2 y2 = pk(rl ? lo(x2) : lo(v2), rh ? hi(x2) : hi(v2));
  const float ql = rl ? lo(nx2) : lo(nv2), qh = rh ? hi(nx2) : hi(nv2);
  const float il = rsqrtf(ql), ih = rsqrtf(qh);
  const F2 inv = pk(lo(y2) < 0.f ? -il : il, hi(y2) < 0.f ? -ih : ih);  // z_b in S^2_+ 
  const F2 n0 = y0 * inv, n1 = y1 * inv, n2 = y2 * inv;
  // kappa = lambda_min / trace (reading R1), lambda_min = Rayleigh quotient of n
  const F2 t0 = fma2(C00, n0, fma2(C01, n1, C02 * n2));
  const F2 t1 = fma2(C01, n0, fma2(C11, n1, C12 * n2));
  const F2 t2 = fma2(C02, n0, fma2(C12, n1, C22 * n2));
  const F2 rq = fma2(n0, t0, fma2(n1, t1, n2 * t2));
  const F2 kap = pk(fmaxf(0.f, lo(rq)) * frcp(lo(tr)), fmaxf(0.f, hi(rq)) * frcp(hi(tr)));
  // Eqs. 2-3 reduced: b3.x_b = -n_z u / |n x x_yaw|, b3.y_b = (n_x sin - n_y cos) / |n x x_yaw|
  const F2 u = fma2(n0, bc(csk.x), n1 * bc(csk.y));
  const F2 t = fma2(n0, bc(csk.y), n1 * bc(-csk.x));
  const F2 w = fma2(n2, n2, t * t);
  const F2 rs = pk(rsqrtf(lo(w)), rsqrtf(hi(w)));
  const F2 spv = (n2 * u) * (rs * bc(-1.f));
  const F2 srv = t * rs;
  const F2 sp = pk(fminf(1.f, fmaxf(-1.f, lo(spv))), fminf(1.f, fmaxf(-1.f, hi(spv))));
  const F2 sr = pk(fminf(1.f, fmaxf(-1.f, lo(srv))), fminf(1.f, fmaxf(-1.f, hi(srv))));
  const F2 pitch = asin2(sp), roll = asin2(sr);
  const F2 ax = pk(fabsf(lo(pitch)), fabsf(hi(pitch))), ay = pk(fabsf(lo(roll)), fabsf(hi(roll)));
  const F2 rk = fma2(bc(p.wk), kap, fma2(bc(p.wx), ax, ay * bc(p.wy)));
  const bool el = lo(kap) > p.kappa_max || lo(ax) > p.phi_x_max || lo(ay) > p.phi_y_max;
  const bool eh = hi(kap) > p.kappa_max || hi(ax) > p.phi_x_max || hi(ay) > p.phi_y_max;
  const bool vl = okl && lo(n2) > 0.f, vh = okh && hi(n2) > 0.f;  // valid normal (reading R11)
  const float qn = __int_as_float(0x7fc00000);
  StateOut2 o;
  o.risk = pk((vl && !el) ? lo(rk) : 1.f, (vh && !eh) ? hi(rk) : 1.f);
  o.pitch = pk(vl ? lo(pitch) : qn, vh ? hi(pitch) : qn);
  o.roll = pk(vl ? lo(roll) : qn, vh ? hi(roll) : qn);
  const F2 zz = bc(href) + mh;  // unclipped: the fitted plane passes through the footprint mean (R14)
  o.z = pk(vl ? lo(zz) : qn, vh ? hi(zz) : qn);
  o.trav_a = (vl && !el) ? 1u : 0u;
  o.trav_b = (vh && !eh) ? 1u : 0u;
  return o;
}

// ------------------------------------------------------------------------------------------
// The assess kernel.
// ------------------------------------------------------------------------------------------
template <int R_T>
struct Geom {
  static constexpr int TY = tile_rows(R_T);
  static constexpr int RPW = TY / NWARPS;    // tile rows (states) per thread per yaw bin
  static constexpr int HX = TX + 2 * R_T;    // halo width (cells)
  static constexpr int HY = TY + 2 * R_T;    // halo height
  static constexpr int PW = HX + 1;          // prefix row length (exclusive prefix, entry 0 = 0)
  static constexpr int NR = 2 * R_T + 1;     // stencil rows
  static constexpr int CPL = (HX + 31) / 32;  // halo cells per lane in the row scan
  static constexpr size_t raw_bytes = ((size_t)HX * HY * 4 + 127) / 128 * 128;
  static constexpr size_t p02_off = raw_bytes;                              // float2 {P0, P2}
  static constexpr size_t px_off = p02_off + (size_t)HY * PW * 8;           // float  PX
  static constexpr size_t pv_off = px_off + (size_t)HY * PW * 4;            // float2 {PV, PVX}
  static constexpr size_t pvxx_off = pv_off + (size_t)HY * PW * 8;          // float  PVXX
  static constexpr size_t misc_off = (pvxx_off + (size_t)HY * PW * 4 + 15) / 16 * 16;
  static constexpr size_t runs_off = misc_off + 128;  // int4 byte offsets per (bin, stencil row)
  static size_t bytes(int k_chunk) { return runs_off + (size_t)k_chunk * NR * 16; }
};

template <int R_T>
__global__ void __launch_bounds__(NTHREADS, 2)
    assess_kernel(const AssessParams p, const __grid_constant__ CUtensorMap tmap) {
  using G = Geom<R_T>;
  constexpr int HX = G::HX, HY = G::HY, PW = G::PW, NR = G::NR, CPL = G::CPL, TY = G::TY, RPW = G::RPW;
  extern __shared__ __align__(128) unsigned char smem[];
  float* raw = reinterpret_cast<float*>(smem);
  float2* p02 = reinterpret_cast<float2*>(smem + G::p02_off);
  float* pxh = reinterpret_cast<float*>(smem + G::px_off);
  float2* pv = reinterpret_cast<float2*>(smem + G::pv_off);
  float* pvxx = reinterpret_cast<float*>(smem + G::pvxx_off);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::misc_off);
  float* red = reinterpret_cast<float*>(smem + G::misc_off + 16);  // [3][8]
  int4* runs_s = reinterpret_cast<int4*>(smem + G::runs_off);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx_rel = (int)(blockIdx.x % (unsigned)p.tiles_x);
  const int ty_rel = p.row_first + (int)(blockIdx.x / (unsigned)p.tiles_x) * p.row_mod;
  if (p.n_rects) {  // INCREMENTAL: only tiles that hold a state within R of a changed cell (CTA-uniform exit)
    bool hit = false;
    for (int q = 0; q < p.n_rects; ++q)
      hit |= tx_rel >= p.rects[q].x && tx_rel < p.rects[q].y && ty_rel >= p.rects[q].z && ty_rel < p.rects[q].w;
    if (!hit) return;
  }
  const long long TI = p.TI0 + tx_rel;
  const long long TJ = p.TJ0 + ty_rel;
  const long long li0 = TI * TX - R_T - p.I_M;  // logical (window) index of halo column 0
  const long long lj0 = TJ * TY - R_T - p.J_M;
  const int kb = p.k_begin + blockIdx.y * p.k_chunk;
  const int ke = min(kb + p.k_chunk, p.k_end);
  if (kb >= ke) return;

  // ---- 1. halo -> shared memory ----------------------------------------------------------
  const bool box_in = li0 >= 0 && li0 + HX <= p.nx && lj0 >= 0 && lj0 + HY <= p.ny;
  int bx = 0, by = 0;
  if (box_in) {
    bx = p.pxM + (int)li0; if (bx >= p.nx) bx -= p.nx;
    by = p.pyM + (int)lj0; if (by >= p.ny) by -= p.ny;
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
        int px = p.pxM + (int)li; if (px >= p.nx) px -= p.nx;
        int py = p.pyM + (int)lj; if (py >= p.ny) py -= p.ny;
        v = __ldg(p.h + (size_t)py * p.ldh + px);
      }
      raw[idx] = v;
    }
  }
  // non-empty stencil rows of this CTA's bins (compacted on the host) as byte offsets into the prefix
  // arrays: (8*ea, 8*eb, 4*ea, dj) with ea = halo index of (row d, column R_T + a), eb = (d, R_T + b + 1)
  for (int idx = tid; idx < (ke - kb) * NR; idx += NTHREADS) {
    const int4 ab = p.runs[(size_t)kb * NR + idx];  // (a, b, d, -)
    const int ea = ab.z * PW + R_T + ab.x, eb = ab.z * PW + R_T + ab.y + 1;
    runs_s[idx] = make_int4(ea * 8, eb * 8, ea * 4, __float_as_int((float)(ab.z - R_T)));
  }
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
  for (int w = 1; w < NWARPS; ++w) { mn = fminf(mn, red[w]); mxv = fmaxf(mxv, red[8 + w]); allvf = fminf(allvf, red[16 + w]); }
  const bool fast = allvf > 0.5f && !p.force_general;
  const float href = (mn <= mxv) ? 0.5f * (mn + mxv) : 0.f;

  // ---- 3. per-row exclusive prefix sums (warp w: rows w, w+8, ...) ---------------------------
  constexpr float XC = (float)(R_T + TX / 2);  // x' = col - XC; the state at lane l has x' = l - TX/2
  for (int row = warp; row < HY; row += NWARPS) {
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
  const long long li = TI * TX + lane - p.I_M;
  const bool col_in = li >= 0 && li < p.nx;
  int pxs = 0;
  if (col_in) { pxs = p.pxM + (int)li; if (pxs >= p.nx) pxs -= p.nx; }
  const bool col_any = __any_sync(0xffffffffu, col_in);
  int off[RPW], pys[RPW];
  bool in[RPW];
#pragma unroll
  for (int s = 0; s < RPW; ++s) {
    const long long lj = TJ * TY + warp + s * NWARPS - p.J_M;
    const bool row_in = lj >= 0 && lj < p.ny;
    in[s] = col_in && row_in;
    int py = 0;
    if (row_in) { py = p.pyM + (int)lj; if (py >= p.ny) py -= p.ny; }
    pys[s] = row_in ? py : -1;
    off[s] = py * p.nx + pxs;
  }
  const int gword = (int)(((TI % p.trav_words) + p.trav_words) % p.trav_words);  // floor(I/32) = TI
  // per-thread byte bases of the prefix arrays at (halo row = tile row of state 0, column lane)
  const char* b8 = reinterpret_cast<const char*>(p02) + (size_t)(warp * PW + lane) * 8;
  const char* b4 = reinterpret_cast<const char*>(pxh) + (size_t)(warp * PW + lane) * 4;
  const char* bv8 = reinterpret_cast<const char*>(pv) + (size_t)(warp * PW + lane) * 8;
  const char* bv4 = reinterpret_cast<const char*>(pvxx) + (size_t)(warp * PW + lane) * 4;
  constexpr int RS8 = NWARPS * PW * 8, RS4 = NWARPS * PW * 4;  // state s -> s * NWARPS halo rows lower

  for (int k = kb; k < ke; ++k) {
    const int4* rk = runs_s + (k - kb) * NR;
    const int nr = __ldg(p.nrows + k);
    const float4 g = __ldg(p.geo + k);
    const float2 csk = __ldg(p.cs + k);
    float2 S02[RPW];
    float SXH[RPW], SYH[RPW];
    float N[RPW], Sx[RPW], Sy[RPW], Sxx[RPW], Sxy[RPW], Syy[RPW];
#pragma unroll
    for (int s = 0; s < RPW; ++s) {
      S02[s] = make_float2(0.f, 0.f);
      SXH[s] = SYH[s] = 0.f;
      N[s] = g.x; Sx[s] = 0.f; Sy[s] = 0.f; Sxx[s] = g.y; Sxy[s] = g.z; Syy[s] = g.w;
    }
    if (fast) {
#pragma unroll 2
      for (int d = 0; d < nr; ++d) {
        const int4 o = rk[d];
        const float dj = __int_as_float(o.w);
        const char* pa8 = b8 + o.x;
        const char* pb8 = b8 + o.y;
        const char* pa4 = b4 + o.z;
        const char* pb4 = b4 + (o.z + ((o.y - o.x) >> 1));
#pragma unroll
        for (int s = 0; s < RPW; ++s) {
          const float2 A = *reinterpret_cast<const float2*>(pa8 + s * RS8);
          const float2 B = *reinterpret_cast<const float2*>(pb8 + s * RS8);
          const float ax = *reinterpret_cast<const float*>(pa4 + s * RS4);
          const float bxv = *reinterpret_cast<const float*>(pb4 + s * RS4);
          const float2 dd = sub2(B, A);  // (run sum of h^, run sum of h^2)
          S02[s] = add2(S02[s], dd);
          SXH[s] += fmaf(-xs, dd.x, bxv - ax);
          SYH[s] = fmaf(dj, dd.x, SYH[s]);
        }
      }
    } else {
#pragma unroll
      for (int s = 0; s < RPW; ++s) { N[s] = Sxx[s] = Sxy[s] = Syy[s] = 0.f; }
#pragma unroll 1
      for (int d = 0; d < nr; ++d) {
        const int4 o = rk[d];
        const float dj = __int_as_float(o.w);
        const int ob4 = o.z + ((o.y - o.x) >> 1);
#pragma unroll
        for (int s = 0; s < RPW; ++s) {
          const float2 A = *reinterpret_cast<const float2*>(b8 + o.x + s * RS8);
          const float2 B = *reinterpret_cast<const float2*>(b8 + o.y + s * RS8);
          const float ax = *reinterpret_cast<const float*>(b4 + o.z + s * RS4);
          const float bxv = *reinterpret_cast<const float*>(b4 + ob4 + s * RS4);
          const float2 VA = *reinterpret_cast<const float2*>(bv8 + o.x + s * RS8);
          const float2 VB = *reinterpret_cast<const float2*>(bv8 + o.y + s * RS8);
          const float wa = *reinterpret_cast<const float*>(bv4 + o.z + s * RS4);
          const float wb = *reinterpret_cast<const float*>(bv4 + ob4 + s * RS4);
          const float2 dd = sub2(B, A);
          const float cnt = VB.x - VA.x, sxv = VB.y - VA.y, sxxv = wb - wa;  // exact integers
          const float sdi = fmaf(-xs, cnt, sxv);                              // sum di over the run
          S02[s] = add2(S02[s], dd);
          SXH[s] += fmaf(-xs, dd.x, bxv - ax);
          SYH[s] = fmaf(dj, dd.x, SYH[s]);
          N[s] += cnt;
          Sx[s] += sdi;
          Sxx[s] += fmaf(xs * xs, cnt, fmaf(-2.f * xs, sxv, sxxv));
          Sy[s] = fmaf(dj, cnt, Sy[s]);
          Syy[s] = fmaf(dj * dj, cnt, Syy[s]);
          Sxy[s] = fmaf(dj, sdi, Sxy[s]);
        }
      }
    }
    float4* outk = p.out + (size_t)k * plane;
    float4* outk2 = p.out + (size_t)(k + p.H) * plane;
    uint32_t* travk = p.trav + (size_t)k * p.ny * p.trav_words + gword;
    uint32_t* travk2 = p.trav + (size_t)(k + p.H) * p.ny * p.trav_words + gword;
    auto store = [&](int s, float risk, float pitch, float roll, float z, unsigned trav) {
      if (in[s]) {
        outk[off[s]] = make_float4(risk, pitch, roll, z);
        if (p.paired) outk2[off[s]] = make_float4(risk, -pitch, -roll, z);
      }
      // traversable bits: the warp's 32 lanes are one world-aligned 32-group = one word
      const unsigned tmask = __ballot_sync(0xffffffffu, in[s] && trav);
      if (lane == 0 && col_any && pys[s] >= 0) {
        travk[(size_t)pys[s] * p.trav_words] = tmask;
        if (p.paired) travk2[(size_t)pys[s] * p.trav_words] = tmask;
      }
    };
    if (fast) {
      const float4 gc = __ldg(p.geoc + 2 * k), gd = __ldg(p.geoc + 2 * k + 1);
#pragma unroll
      for (int s = 0; s < RPW; s += 2) {
        const StateOut2 o = epilogue2(pk(S02[s].x, S02[s + 1].x), pk(S02[s].y, S02[s + 1].y), pk(SXH[s], SXH[s + 1]),
                                      pk(SYH[s], SYH[s + 1]), href, gc, gd, csk, p);
        store(s, lo(o.risk), lo(o.pitch), lo(o.roll), lo(o.z), o.trav_a);
        store(s + 1, hi(o.risk), hi(o.pitch), hi(o.roll), hi(o.z), o.trav_b);
      }
    } else {
#pragma unroll
      for (int s = 0; s < RPW; ++s) {
        const StateOut o = epilogue(N[s], Sx[s], Sy[s], Sxx[s], Sxy[s], Syy[s], S02[s].x, S02[s].y, SXH[s], SYH[s],
                                    href, csk, p, true);
        store(s, o.risk, o.pitch, o.roll, o.z, (unsigned)o.trav);
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

__device__ __forceinline__ long long floor_div32(long long a) { return a >= 0 ? a / 32 : -((-a + 31) / 32); }

__global__ void gather_logical_kernel(const AssessParams p, int k_lo, int k_hi, float* risk, float* pitch,
                                      float* roll, float* z, uint8_t* trav) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i >= p.nx) return;
  int px = p.pxM + i; if (px >= p.nx) px -= p.nx;
  int py = p.pyM + j; if (py >= p.ny) py -= p.ny;
  const size_t src = ((size_t)k * p.ny + py) * p.nx + px;
  const size_t dst = ((size_t)k * p.ny + j) * p.nx + i;
  const bool owned = k >= k_lo && k < k_hi;
  const float qnan = __int_as_float(0x7fc00000);
  const float4 v = owned ? p.out[src] : make_float4(qnan, qnan, qnan, qnan);
  if (risk) risk[dst] = v.x;
  if (pitch) pitch[dst] = v.y;
  if (roll) roll[dst] = v.z;
  if (z) z[dst] = v.w;
  if (trav) {
    const long long I = p.I_M + i;
    const long long gw = floor_div32(I);
    const int w = (int)(((gw % p.trav_words) + p.trav_words) % p.trav_words);
    const int bit = (int)(I - gw * 32);
    trav[dst] = owned ? (uint8_t)((p.trav[((size_t)k * p.ny + py) * p.trav_words + w] >> bit) & 1u) : 0;
  }
}

cudaError_t launch_gather_logical(const AssessParams& p, int k_lo, int k_hi, float* risk, float* pitch, float* roll,
                                  float* z, uint8_t* trav, cudaStream_t s) {
  dim3 grid((p.nx + 255) / 256, p.ny, p.n_yaw);
  gather_logical_kernel<<<grid, 256, 0, s>>>(p, k_lo, k_hi, risk, pitch, roll, z, trav);
  return cudaGetLastError();
}

__global__ void query_kernel(const AssessParams p, int n, const int4* __restrict__ idx, float* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int4 e = idx[q];
  const float qnan = __int_as_float(0x7fc00000);
  float4 v = make_float4(qnan, qnan, qnan, qnan);
  float tv = 0.f;
  if (e.w) {
    v = p.out[((size_t)e.z * p.ny + e.y) * p.nx + e.x];
    const int wb = e.w - 1;
    tv = (float)((p.trav[((size_t)e.z * p.ny + e.y) * p.trav_words + (wb >> 5)] >> (wb & 31)) & 1u);
  }
  out[q] = v.x; out[n + q] = v.y; out[2 * (size_t)n + q] = v.z; out[3 * (size_t)n + q] = v.w; out[4 * (size_t)n + q] = tv;
}

cudaError_t launch_query(const AssessParams& p, int n, const int4* idx, float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  query_kernel<<<(n + 255) / 256, 256, 0, s>>>(p, n, idx, out);
  return cudaGetLastError();
}

}  // namespace se2m
