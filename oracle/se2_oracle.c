/*
 * se2_oracle.c — plain, slow, FP64 CPU oracle for the SE(2) traversability hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2503_02412_b200/),
 * and it never reads anything the CUDA path produced.
 *
 * What it computes: Algorithm 1 of the paper (§V.B, "Traversability
 * and terrain pose mapping assessment in state s_r in SE(2)") for one state at a time,
 * step by step in the paper's order, in IEEE double, with no blocking, fusion or
 * precomputed tables:
 *   line 1  FindEllipticalPoints   -> gather_points()
 *   line 2  GetMeanPosition   -> mean of the gathered points
 *   lines 3-8 covariance, /NumOf(P) -> two-pass sum of p_e p_e^T / N
 *   line 9  GetMinEigenVecWithCurv   -> cyclic Jacobi (orc_eig3), kappa
 *   lines 10-11 kappa test
 *   line 12 GetXbYb                (Eqs. 2-3)
 *   line 13 phi_x, phi_y
 *   lines 14-18 attitude test, weighted risk
 * Readings of what the paper leaves open are the DESIGN.md readings R1..R21 (= SURVEY.md
 * §8(c) C1..C21); each is cited where it is applied.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared -o liboracle.so se2_oracle.c -lm -lpthread
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t nx, ny;        /* window cells; x = columns (fastest) */
  int32_t n_yaw;         /* yaw bins over [-pi, pi) (reading R3) */
  int32_t pad0;
  double resolution;     /* l_res, m per cell (Eq. 4) */
  double ex, ey;         /* ellipse semi-axes (m), e_x along x_yaw (reading R4) */
  double w[3];           /* w_r (Alg. 1 input) */
  double kappa_max;      /* kappa_max */
  double phi_x_max;      /* phi_x,max (0.52 rad) */
  double phi_y_max;      /* phi_y,max */
} orc_params;

typedef struct {
  double risk, pitch, roll, z, kappa, gap;
  double lam[3];         /* ascending eigenvalues of Cov */
  double n[3];           /* z_b: unit eigenvector of lam[0], n_z > 0 */
  int32_t trav;          /* 1 = traversable (no early return, not unknown) (reading R17) */
  int32_t status;        /* 0 ok, 1 unknown (N < 3), 2 degenerate covariance (reading R11) */
  int32_t n_points;      /* |P| */
  int32_t early;         /* 0 none, 1 kappa > kappa_max, 2 attitude limit */
} orc_result;

/* ---------------------------------------------------------------------------------- */
/* 3x3 symmetric eigen-decomposition by the cyclic Jacobi method (Golub & Van Loan,     */
/* Matrix Computations, Alg. 8.4.3).  Textbook, deliberately not the GPU's algorithm.   */
/* A (row-major 3x3) is symmetric.  Output: lam ascending, V columns = eigenvectors.     */
/* ---------------------------------------------------------------------------------- */
int orc_eig3(const double* Ain, double* lam, double* Vout) {
  double A[3][3], V[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      A[r][c] = Ain[3 * r + c];
      V[r][c] = (r == c) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, fro = 0.0;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        fro += A[r][c] * A[r][c];
        if (r != c) off += A[r][c] * A[r][c];
      }
    if (off == 0.0 || sqrt(off) <= 1e-15 * sqrt(fro)) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        /* symmetric Schur decomposition of the (p,q) 2x2 block (GVL Alg. 8.4.1) */
        double tau = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        double t;
        if (fabs(tau) > 1e150)
          t = 0.5 / tau;
        else
          t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = t * c;
        /* J = identity except J[p][p]=c, J[p][q]=s, J[q][p]=-s, J[q][q]=c.  A <- J^T A J, V <- V J. */
        double J[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
        J[p][p] = c; J[p][q] = s; J[q][p] = -s; J[q][q] = c;
        double T[3][3], B[3][3], W[3][3];
        for (int r = 0; r < 3; ++r)
          for (int cc = 0; cc < 3; ++cc) {
            double acc = 0.0;
            for (int m = 0; m < 3; ++m) acc += A[r][m] * J[m][cc];
            T[r][cc] = acc;
          }
        for (int r = 0; r < 3; ++r)
          for (int cc = 0; cc < 3; ++cc) {
            double acc = 0.0;
            for (int m = 0; m < 3; ++m) acc += J[m][r] * T[m][cc];
            B[r][cc] = acc;
          }
        for (int r = 0; r < 3; ++r)
          for (int cc = 0; cc < 3; ++cc) {
            double acc = 0.0;
            for (int m = 0; m < 3; ++m) acc += V[r][m] * J[m][cc];
            W[r][cc] = acc;
          }
        memcpy(A, B, sizeof A);
        memcpy(V, W, sizeof V);
      }
  }
  /* sort ascending (selection sort over 3 entries) */
  int idx[3] = {0, 1, 2};
  double d[3] = {A[0][0], A[1][1], A[2][2]};
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b)
      if (d[idx[b]] < d[idx[a]]) { int tmp = idx[a]; idx[a] = idx[b]; idx[b] = tmp; }
  for (int m = 0; m < 3; ++m) {
    lam[m] = d[idx[m]];
    for (int r = 0; r < 3; ++r) Vout[3 * r + m] = V[r][idx[m]];
  }
  return 0;
}

/* ---------------------------------------------------------------------------------- */
/* Algorithm 1, one state.                                                              */
/* ---------------------------------------------------------------------------------- */
static double theta_of_bin(int k, int n_yaw) {
  /* reading R3: theta_k = -pi + 2*pi*k/n_yaw over [-pi, pi) */
  return -M_PI + 2.0 * M_PI * (double)k / (double)n_yaw;
}

static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* FindEllipticalPoints (Alg. 1 line 1).  Reading R5: cell centres, q in cell
 * units with the representative angle theta'_k (the ellipse depends on theta mod pi),
 * include iff q <= 1 + 1e-9.  Reading R6: points in state-local metric coordinates
 * (di*r, dj*r, h) with absolute heights.  Readings R8/R9: only cells inside the window
 * and known.  Returns |P|; pts has room for (2R+1)^2 points. */
static int gather_points(const orc_params* P, const float* h, const uint8_t* known, int i, int j,
                         int k, double* pts) {
  const double r = P->resolution;
  const double a = P->ex / r, b = P->ey / r;
  int krep = k;
  if (P->n_yaw % 2 == 0) krep = k % (P->n_yaw / 2);
  const double th = theta_of_bin(krep, P->n_yaw);
  const double c = cos(th), s = sin(th);
  const int R = (int)ceil(fmax(a, b)) + 1;
  int n = 0;
  for (int dj = -R; dj <= R; ++dj)
    for (int di = -R; di <= R; ++di) {
      const double u = di * c + dj * s;   /* along x_yaw */
      const double v = -di * s + dj * c;  /* along y_yaw */
      const double q = (u / a) * (u / a) + (v / b) * (v / b);
      if (!(q <= 1.0 + 1e-9)) continue;
      const int ii = i + di, jj = j + dj;
      if (ii < 0 || ii >= P->nx || jj < 0 || jj >= P->ny) continue;
      const size_t cell = (size_t)jj * (size_t)P->nx + (size_t)ii;
      if (known && !known[cell]) continue;
      pts[3 * n + 0] = di * r;
      pts[3 * n + 1] = dj * r;
      pts[3 * n + 2] = (double)h[cell];
      ++n;
    }
  return n;
}

int orc_assess_state_ex(const orc_params* P, const float* h, const uint8_t* known, int i, int j, int k,
                        uint64_t shuffle_seed, double* scratch, orc_result* out) {
  memset(out, 0, sizeof *out);
  const double nan = NAN;
  /* line 1: P <- FindEllipticalPoints(M, s_r, e_x, e_y) */
  const int N = gather_points(P, h, known, i, j, k, scratch);
  out->n_points = N;
  if (shuffle_seed) { /* test hook for pin Q8 (tap-order invariance): Fisher-Yates */
    uint64_t st = shuffle_seed;
    for (int m = N - 1; m > 0; --m) {
      int o = (int)(splitmix64(&st) % (uint64_t)(m + 1));
      for (int c = 0; c < 3; ++c) { double t = scratch[3 * m + c]; scratch[3 * m + c] = scratch[3 * o + c]; scratch[3 * o + c] = t; }
    }
  }
  if (N < 3) { /* SPEC S:234 "fewer than 3 points -> unknown-risk"; reading R8 */
    out->risk = 1.0; out->pitch = out->roll = out->z = out->kappa = out->gap = nan;
    out->lam[0] = out->lam[1] = out->lam[2] = nan;
    out->n[0] = out->n[1] = out->n[2] = nan;
    out->trav = 0; out->status = 1;
    return 0;
  }
  /* line 2: p_mean <- GetMeanPosition(P) */
  double m[3] = {0.0, 0.0, 0.0};
  for (int p = 0; p < N; ++p)
    for (int c = 0; c < 3; ++c) m[c] += scratch[3 * p + c];
  for (int c = 0; c < 3; ++c) m[c] /= (double)N;
  /* lines 3-8: Cov <- sum (p_j - p_mean)(p_j - p_mean)^T ; line 8: Cov <- Cov / NumOf(P) */
  double C[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = 0; p < N; ++p) {
    double e[3];
    for (int c = 0; c < 3; ++c) e[c] = scratch[3 * p + c] - m[c];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) C[3 * r + c] += e[r] * e[c];
  }
  for (int q = 0; q < 9; ++q) C[q] /= (double)N;
  /* line 9: z_b, kappa_ter <- GetMinEigenVecWithCurv(Cov) */
  double lam[3], V[9];
  orc_eig3(C, lam, V);
  double n[3] = {V[0], V[3], V[6]};                 /* eigenvector of lam[0] */
  if (n[2] < 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; } /* S^2_+  */
  if (lam[0] < 0.0) lam[0] = 0.0;                   /* Cov is PSD; reading R1 (rounding) */
  const double tr = lam[0] + lam[1] + lam[2];
  for (int c = 0; c < 3; ++c) { out->lam[c] = lam[c]; out->n[c] = n[c]; }
  if (!(lam[1] - lam[0] > 1e-12 * tr) || !(n[2] > 1e-12)) { /* reading R11: degenerate */
    out->risk = 1.0; out->pitch = out->roll = out->z = out->kappa = out->gap = nan;
    out->trav = 0; out->status = 2;
    return 0;
  }
  const double kappa = lam[0] / tr;                 /* reading R1: surface variation */
  out->kappa = kappa;
  out->gap = (lam[2] > 0.0) ? (lam[1] - lam[0]) / lam[2] : 0.0;
  /* z = f_1(x, y, theta): height of the fitted plane at the state centre (reading R14) */
  out->z = m[2] + (n[0] * m[0] + n[1] * m[1]) / n[2];
  /* line 12: x_b, y_b <- GetXbYb(z_b, s_r)  (Eqs. 2-3) */
  double xyaw[3];
  if (P->n_yaw % 2 == 0 && k >= P->n_yaw / 2) {     /* exact negation of bin k - n/2 (reading R3) */
    const double th = theta_of_bin(k - P->n_yaw / 2, P->n_yaw);
    xyaw[0] = -cos(th); xyaw[1] = -sin(th); xyaw[2] = 0.0;
  } else {
    const double th = theta_of_bin(k, P->n_yaw);
    xyaw[0] = cos(th); xyaw[1] = sin(th); xyaw[2] = 0.0;
  }
  double cyb[3] = {n[1] * xyaw[2] - n[2] * xyaw[1], n[2] * xyaw[0] - n[0] * xyaw[2],
                   n[0] * xyaw[1] - n[1] * xyaw[0]};              /* z_b x x_yaw */
  const double cn = sqrt(cyb[0] * cyb[0] + cyb[1] * cyb[1] + cyb[2] * cyb[2]);
  double yb[3] = {cyb[0] / cn, cyb[1] / cn, cyb[2] / cn};        /* Eq. 2 */
  double xb[3] = {yb[1] * n[2] - yb[2] * n[1], yb[2] * n[0] - yb[0] * n[2],
                  yb[0] * n[1] - yb[1] * n[0]};                   /* Eq. 3: y_b x z_b */
  /* line 13: phi = |asin(b3^T x_b)|, |asin(b3^T y_b)|; signed values stored (reading R13) */
  const double sx = fmin(1.0, fmax(-1.0, xb[2]));
  const double sy = fmin(1.0, fmax(-1.0, yb[2]));
  out->pitch = asin(sx);
  out->roll = asin(sy);
  const double phix = fabs(out->pitch), phiy = fabs(out->roll);
  /* lines 10-11: if kappa > kappa_max return (1, z_b)  (strict, reading R15) */
  if (kappa > P->kappa_max) { out->risk = 1.0; out->trav = 0; out->early = 1; return 0; }
  /* lines 14-15: attitude limits */
  if (phix > P->phi_x_max || phiy > P->phi_y_max) { out->risk = 1.0; out->trav = 0; out->early = 2; return 0; }
  /* lines 16-17: r = [kappa/kappa_max, phi_x/phi_x_max, phi_y/phi_y_max]; Risk = r^T w_r */
  const double rv[3] = {kappa / P->kappa_max, phix / P->phi_x_max, phiy / P->phi_y_max};
  out->risk = rv[0] * P->w[0] + rv[1] * P->w[1] + rv[2] * P->w[2];
  out->trav = 1;
  return 0;
}

static int max_points(const orc_params* P) {
  const double a = P->ex / P->resolution, b = P->ey / P->resolution;
  const int R = (int)ceil(fmax(a, b)) + 1;
  return (2 * R + 1) * (2 * R + 1);
}

int orc_assess_state(const orc_params* P, const float* h, const uint8_t* known, int i, int j, int k,
                     uint64_t shuffle_seed, orc_result* out) {
  double* scratch = (double*)malloc(sizeof(double) * 3 * (size_t)max_points(P));
  if (!scratch) return -1;
  int rc = orc_assess_state_ex(P, h, known, i, j, k, shuffle_seed, scratch, out);
  free(scratch);
  return rc;
}

/* ---------------------------------------------------------------------------------- */
/* Many states: a static partition of the state list over POSIX threads.  Each state's  */
/* arithmetic is sequential, so results do not depend on the thread count.              */
/* ---------------------------------------------------------------------------------- */
typedef struct {
  const orc_params* P;
  const float* h;
  const uint8_t* known;
  const int32_t* ijk;   /* n x 3, or NULL = all states in [k][j][i] order */
  int64_t begin, end;
  orc_result* out;
  int rc;
} orc_job;

static void* orc_worker(void* arg) {
  orc_job* J = (orc_job*)arg;
  double* scratch = (double*)malloc(sizeof(double) * 3 * (size_t)max_points(J->P));
  if (!scratch) { J->rc = -1; return NULL; }
  const int64_t plane = (int64_t)J->P->nx * J->P->ny;
  for (int64_t s = J->begin; s < J->end; ++s) {
    int i, j, k;
    if (J->ijk) { i = J->ijk[3 * s]; j = J->ijk[3 * s + 1]; k = J->ijk[3 * s + 2]; }
    else { k = (int)(s / plane); j = (int)((s % plane) / J->P->nx); i = (int)(s % J->P->nx); }
    orc_assess_state_ex(J->P, J->h, J->known, i, j, k, 0, scratch, &J->out[s]);
  }
  free(scratch);
  J->rc = 0;
  return NULL;
}

static int validate(const orc_params* P) {
  if (!P || P->nx < 1 || P->ny < 1 || P->n_yaw < 1) return -2;
  if (!(P->resolution > 0) || !(P->ex > 0) || !(P->ey > 0)) return -2;
  if (!(P->kappa_max > 0) || !(P->phi_x_max > 0) || !(P->phi_y_max > 0)) return -2;
  return 0;
}

/* ijk == NULL: all n_yaw*ny*nx states, out in [k][j][i] order (n is ignored). */
int orc_assess_states(const orc_params* P, const float* h, const uint8_t* known, int64_t n,
                      const int32_t* ijk, orc_result* out, int nthreads) {
  int rc = validate(P);
  if (rc) return rc;
  if (!ijk) n = (int64_t)P->nx * P->ny * P->n_yaw;
  if (ijk)
    for (int64_t s = 0; s < n; ++s)
      if (ijk[3 * s] < 0 || ijk[3 * s] >= P->nx || ijk[3 * s + 1] < 0 || ijk[3 * s + 1] >= P->ny ||
          ijk[3 * s + 2] < 0 || ijk[3 * s + 2] >= P->n_yaw)
        return -3;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((int64_t)nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  orc_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].P = P; jobs[t].h = h; jobs[t].known = known; jobs[t].ijk = ijk; jobs[t].out = out;
    jobs[t].begin = n * t / nthreads; jobs[t].end = n * (t + 1) / nthreads; jobs[t].rc = 0;
  }
  if (nthreads == 1) { orc_worker(&jobs[0]); return jobs[0].rc; }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, orc_worker, &jobs[t]);
  rc = 0;
  for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); if (jobs[t].rc) rc = jobs[t].rc; }
  return rc;
}

int orc_result_size(void) { return (int)sizeof(orc_result); }
int orc_params_size(void) { return (int)sizeof(orc_params); }

/* ---------------------------------------------------------------------------------- */
/* Signed distance field of one yaw layer (NEXT-2; "the corresponding signed  */
/* distance field (SDF) will be generated", "the distance to the edge of the  */
/* nearest region, with negative values inside obstacles").  Reading R24:    */
/* obstacle = Risk = 1; a free cell's value is the Euclidean distance (m)   */
/* between cell centres to the nearest obstacle cell, an obstacle cell's value is minus    */
/* the distance to the nearest free cell; distances are clamped to [-d_max, d_max]; cells  */
/* with no counterpart in the window get +-d_max.  Brute force over all cell pairs.        */
/* obstacle: ny*nx bytes (1 obstacle, 0 free), row-major, x fastest.                       */
/* ---------------------------------------------------------------------------------- */
typedef struct {
  const uint8_t* obstacle;
  int nx, ny;
  double r, d_max;
  double* out;
  int j_begin, j_end;
} orc_sdf_job;

static void* orc_sdf_worker(void* arg) {
  orc_sdf_job* J = (orc_sdf_job*)arg;
  for (int j = J->j_begin; j < J->j_end; ++j)
    for (int i = 0; i < J->nx; ++i) {
      const int self = J->obstacle[(size_t)j * J->nx + i] ? 1 : 0;
      double best = INFINITY;
      for (int jj = 0; jj < J->ny; ++jj)
        for (int ii = 0; ii < J->nx; ++ii) {
          const int other = J->obstacle[(size_t)jj * J->nx + ii] ? 1 : 0;
          if (other == self) continue;  /* free cell: nearest obstacle; obstacle: nearest free */
          const double dx = (ii - i) * J->r, dy = (jj - j) * J->r;
          const double d = sqrt(dx * dx + dy * dy);
          if (d < best) best = d;
        }
      if (best > J->d_max) best = J->d_max;
      J->out[(size_t)j * J->nx + i] = self ? -best : best;
    }
  return NULL;
}

int orc_sdf_layer(const uint8_t* obstacle, int nx, int ny, double r, double d_max, double* out, int nthreads) {
  if (!obstacle || !out || nx < 1 || ny < 1 || !(r > 0) || !(d_max > 0)) return -2;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads > ny) nthreads = ny;
  pthread_t th[256];
  orc_sdf_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].obstacle = obstacle; jobs[t].nx = nx; jobs[t].ny = ny; jobs[t].r = r; jobs[t].d_max = d_max;
    jobs[t].out = out; jobs[t].j_begin = ny * t / nthreads; jobs[t].j_end = ny * (t + 1) / nthreads;
  }
  if (nthreads == 1) { orc_sdf_worker(&jobs[0]); return 0; }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, orc_sdf_worker, &jobs[t]);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}
