"""FP64 oracle of the elevation-map front-end (NEXT-1) — TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER.md:103-122 (§V.A, Fig. 3), in the paper's order for one frame:
  1. Eq. 4 recentre — ``oracle.Window.shift``;
  2. ray-cast reset: "checking the grid that passes from the LiDAR position to each
     point, setting the state to unknown if the elevation in the grid is higher than the highest value
     predicted by the ray";
  3. point filtering: points outside the map are ignored, the others are transformed to
     the body frame B and points outside a height band are dropped;
  4. the point height z_l and its variance from the Jacobians J_S, J_R, J_B;
  5. 1-D Kalman fusion per cell, multiple points per cell handled by the Mahalanobis distance
     "in the same way as the classical elevation map".
Readings (R26-R30): the world height uses +p_B (the paper's "-p_B" only flips J_B, which
enters sigma^2 quadratically); the height band is on the body-frame z of the point (default +-1.5 m,
SPEC S:164); rays are cast for the filtered points; a traversed cell is one whose open square meets the
open segment, the endpoint's own cell excluded, and its "highest predicted value" is the larger ray
height at the segment's entry / exit of that square, with a margin eps_ray (0.05 m); the
Mahalanobis gate is |z - h| / sqrt(s2 + s2_m) <= 2 and on failure the higher of (z, h) wins
(SPEC S:163); points are fused sequentially in input order; cells store float32 height and variance.

Everything is plain Python / NumPy in float64 with no FMA contraction.

Pinned by tests/test_oracle_frontend.py: the SPEC's worked variance and KF examples, a Monte-Carlo
check of sigma^2, the ray-cast examples, dense sampling of the slab traversal, KF order-insensitivity
and variance monotonicity.  The readings R26-R30 themselves (sign of p_B, band frame, ray geometry,
sequential fusion order, float32 storage) are parity unpinned as readings (not confirmable from the
paper's text).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class FrontendParams:
    z_min: float = -1.5          # body-frame height band (m)
    z_max: float = 1.5
    gate: float = 2.0            # Mahalanobis gate
    ray_eps: float = 0.05        # ray-cast margin (m)


@dataclass
class Pose:
    """Robot pose and the covariances of PAPER.md:106-120."""
    R_B: np.ndarray               # 3x3 body -> world
    p_B: np.ndarray               # 3
    R_BS: np.ndarray = field(default_factory=lambda: np.eye(3))   # sensor -> body
    p_BS: np.ndarray = field(default_factory=lambda: np.zeros(3))  # sensor position in B
    Sigma_S: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))
    Sigma_R: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))
    Sigma_B: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))


def _mv(A, v):
    """3x3 @ 3 written out (fixed summation order)."""
    return [A[0][0] * v[0] + A[0][1] * v[1] + A[0][2] * v[2],
            A[1][0] * v[0] + A[1][1] * v[1] + A[1][2] * v[2],
            A[2][0] * v[0] + A[2][1] * v[1] + A[2][2] * v[2]]


def _quad(v, S):
    """v^T S v written out."""
    Sv = _mv(S, v)
    return v[0] * Sv[0] + v[1] * Sv[1] + v[2] * Sv[2]


def point_measurement(ps, pose: Pose):
    """One sensor-frame point -> (world x, y, z_l, body-frame z, sigma^2)."""
    RB = [[float(pose.R_B[i][j]) for j in range(3)] for i in range(3)]
    RBS = [[float(pose.R_BS[i][j]) for j in range(3)] for i in range(3)]
    q = _mv(RBS, [float(ps[0]), float(ps[1]), float(ps[2])])
    q = [q[0] + float(pose.p_BS[0]), q[1] + float(pose.p_BS[1]), q[2] + float(pose.p_BS[2])]  # point in B
    w = _mv(RB, q)
    w = [w[0] + float(pose.p_B[0]), w[1] + float(pose.p_B[1]), w[2] + float(pose.p_B[2])]     # world
    # J_S = (R_B R_BS)^T b3 : the third row of R_B R_BS
    J_S = [RB[2][0] * RBS[0][k] + RB[2][1] * RBS[1][k] + RB[2][2] * RBS[2][k] for k in range(3)]
    # J_R = q^ R_B^T b3 = q x (third row of R_B)
    t = [RB[2][0], RB[2][1], RB[2][2]]
    J_R = [q[1] * t[2] - q[2] * t[1], q[2] * t[0] - q[0] * t[2], q[0] * t[1] - q[1] * t[0]]
    J_B = [0.0, 0.0, -1.0]
    s2 = _quad(J_S, pose.Sigma_S) + _quad(J_R, pose.Sigma_R) + _quad(J_B, pose.Sigma_B)
    return w[0], w[1], w[2], q[2], max(s2, 0.0)


def _cell_interval(sx, sy, dx, dy, x0, x1, y0, y1):
    """Slab method: parameter interval (t0, t1) of the segment s + t d, t in (0, 1), inside the open
    square (x0, x1) x (y0, y1); None if empty."""
    t0, t1 = 0.0, 1.0
    for s, d, lo, hi in ((sx, dx, x0, x1), (sy, dy, y0, y1)):
        if d == 0.0:
            if not (lo < s < hi):
                return None
            continue
        a, b = (lo - s) / d, (hi - s) / d
        if a > b:
            a, b = b, a
        t0, t1 = max(t0, a), min(t1, b)
    if not (t0 < t1):
        return None
    return t0, t1


def integrate_scan(win, points_s, pose: Pose, P: FrontendParams):
    """One frame on an oracle.Window (its float32 heights / variances and uint8 known arrays are updated
    in place).  Returns per-point status (0 used, 1 outside map,
    2 outside height band, 3 non-positive variance) and the number of cells reset by ray casting."""
    r = win.r
    nx, ny = win.nx, win.ny
    var = win.var
    meas = []
    status = np.zeros(len(points_s), np.int32)
    for n, ps in enumerate(points_s):
        x, y, z, zb, s2 = point_measurement(ps, pose)
        I, J = math.floor(x / r), math.floor(y / r)
        i, j = I - win.I_M, J - win.J_M
        if not (0 <= i < nx and 0 <= j < ny):
            status[n] = 1
            continue
        if not (P.z_min <= zb <= P.z_max):
            status[n] = 2
            continue
        if not (s2 > 0.0):
            status[n] = 3
            continue
        meas.append((n, i, j, x, y, z, s2))
    # ---- 2. ray-cast reset against the heights before this frame's fusion ----
    RB = pose.R_B
    sx = float(RB[0][0] * pose.p_BS[0] + RB[0][1] * pose.p_BS[1] + RB[0][2] * pose.p_BS[2]) + float(pose.p_B[0])
    sy = float(RB[1][0] * pose.p_BS[0] + RB[1][1] * pose.p_BS[1] + RB[1][2] * pose.p_BS[2]) + float(pose.p_B[1])
    sz = float(RB[2][0] * pose.p_BS[0] + RB[2][1] * pose.p_BS[1] + RB[2][2] * pose.p_BS[2]) + float(pose.p_B[2])
    h0 = win.heights.copy()
    k0 = win.known.copy()
    reset = np.zeros((ny, nx), dtype=bool)
    for (n, i_e, j_e, x, y, z, s2) in meas:
        dx, dy, dz = x - sx, y - sy, z - sz
        Ia, Ib = sorted((math.floor(sx / r), math.floor(x / r)))
        Ja, Jb = sorted((math.floor(sy / r), math.floor(y / r)))
        for J in range(Ja, Jb + 1):
            j = J - win.J_M
            if not (0 <= j < ny):
                continue
            for I in range(Ia, Ib + 1):
                i = I - win.I_M
                if not (0 <= i < nx) or (i == i_e and j == j_e) or not k0[j, i]:
                    continue
                iv = _cell_interval(sx, sy, dx, dy, I * r, (I + 1) * r, J * r, (J + 1) * r)
                if iv is None:
                    continue
                zr = max(sz + iv[0] * dz, sz + iv[1] * dz)  # highest ray height over the cell
                if float(h0[j, i]) > zr + P.ray_eps:
                    reset[j, i] = True
    win.known[reset] = 0
    # ---- 5. sequential KF fusion in point order ----
    for (n, i, j, x, y, z, s2) in meas:
        if not win.known[j, i]:
            win.heights[j, i] = np.float32(z)
            var[j, i] = np.float32(s2)
            win.known[j, i] = 1
            continue
        h, sc = float(win.heights[j, i]), float(var[j, i])
        d = abs(z - h) / math.sqrt(sc + s2)
        if d <= P.gate:
            hn = (s2 * h + sc * z) / (sc + s2)
            vn = (sc * s2) / (sc + s2)
        elif z > h:
            hn, vn = z, s2
        else:
            continue
        win.heights[j, i] = np.float32(hn)
        var[j, i] = np.float32(vn)
    return status, int(reset.sum())
