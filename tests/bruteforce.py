"""Independent NumPy brute force of Algorithm 1 (pin Q5) — test code, not product code.

Deliberately written differently from the C oracle so that a slip in either shows up:
  * the footprint test is done in METRES with the state's own heading theta_k (not the
    representative angle, not cell units);
  * mean/covariance by ``np.cov(..., bias=True)`` (divisor N);
  * the eigen-solve by ``np.linalg.eigh`` (LAPACK), not Jacobi;
  * pitch/roll by the reduced closed forms  b3^T x_b = -n_z u / sqrt(1-u^2),
    b3^T y_b = (n_x sin th - n_y cos th) / sqrt(1-u^2), u = n . x_yaw
    (vector triple product applied to Eqs. 2-3), not explicit cross products.
States with a cell within 1e-11 of the membership cut q = 1 + 1e-9 (reading R5) are reported
as ties so callers can skip them (none occur in the configurations tested).
"""
from __future__ import annotations

import math

import numpy as np


def assess_state(h, known, i, j, k, r, n_yaw, ex, ey, w=(0.4, 0.3, 0.3), kappa_max=0.1,
                 phi_x_max=0.52, phi_y_max=0.52):
    ny, nx = h.shape
    th = -math.pi + 2.0 * math.pi * k / n_yaw
    R = int(math.ceil(max(ex, ey) / r)) + 1
    di, dj = np.meshgrid(np.arange(-R, R + 1), np.arange(-R, R + 1), indexing="xy")
    dx, dy = di * r, dj * r
    u = dx * math.cos(th) + dy * math.sin(th)
    v = -dx * math.sin(th) + dy * math.cos(th)
    q = (u / ex) ** 2 + (v / ey) ** 2
    tie = bool(np.any(np.abs(q - (1.0 + 1e-9)) < 1e-11))  # membership within rounding of the cut
    ii, jj = i + di, j + dj
    inside = (q <= 1.0 + 1e-9) & (ii >= 0) & (ii < nx) & (jj >= 0) & (jj < ny)
    ii_c, jj_c = np.clip(ii, 0, nx - 1), np.clip(jj, 0, ny - 1)
    if known is not None:
        inside &= known[jj_c, ii_c].astype(bool)
    pts = np.stack([dx[inside], dy[inside], h[jj_c, ii_c][inside].astype(np.float64)], axis=1)
    out = dict(tie=tie, n_points=len(pts))
    if len(pts) < 3:
        out.update(status=1, risk=1.0, trav=0)
        return out
    C = np.cov(pts.T, bias=True)
    lam, V = np.linalg.eigh(C)
    n = V[:, 0] * (1.0 if V[2, 0] > 0 else -1.0)
    lam0 = max(lam[0], 0.0)
    tr = lam0 + lam[1] + lam[2]
    if not (lam[1] - lam0 > 1e-12 * tr) or not (n[2] > 1e-12):
        out.update(status=2, risk=1.0, trav=0)
        return out
    kappa = lam0 / tr
    c, s = math.cos(th), math.sin(th)
    uu = n[0] * c + n[1] * s
    sx = -n[2] * uu / math.sqrt(1.0 - uu * uu)
    sy = (n[0] * s - n[1] * c) / math.sqrt(1.0 - uu * uu)
    pitch, roll = math.asin(max(-1.0, min(1.0, sx))), math.asin(max(-1.0, min(1.0, sy)))
    m = pts.mean(axis=0)
    z = m[2] + (n[0] * m[0] + n[1] * m[1]) / n[2]
    if kappa > kappa_max or abs(pitch) > phi_x_max or abs(roll) > phi_y_max:
        risk, trav = 1.0, 0
    else:
        risk = w[0] * kappa / kappa_max + w[1] * abs(pitch) / phi_x_max + w[2] * abs(roll) / phi_y_max
        trav = 1
    out.update(status=0, risk=risk, trav=trav, pitch=pitch, roll=roll, z=z, kappa=kappa,
               gap=(lam[1] - lam0) / lam[2])
    return out
