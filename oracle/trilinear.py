"""FP64 oracle of the planner's map access — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:227 (§VI.C): "we adopt trilinear interpolation to obtain the values and gradients of the
function G_c and Risk, where operations on manifold are applied for the handling of SO(2) space".
SPEC S:261-269 (query_trilinear): trilinear over (x, y, theta), theta wrapped cyclically across the
+-pi seam; the gradient is the exact gradient of the interpolant (piecewise constant per cell).

Lattice (readings R3/R6): node (i, j, k) of the window sits at x = (I_M + i + 1/2) r,
y = (J_M + j + 1/2) r, theta_k = -pi + 2 pi k / n.  A query needs its 4 spatial corner nodes inside
the window; otherwise it is out of range.

Pinned by tests/test_oracle_trilinear.py (interpolation of linear fields is exact, node values are
reproduced, the gradient matches finite differences, theta wraps); the lattice placement (R25) is a
reading: parity unpinned as a reading.
"""
from __future__ import annotations

import math

import numpy as np


def trilinear(volume, I_M: int, J_M: int, r: float, xyt):
    """volume: [n_yaw][ny][nx] float array; xyt: (n, 3) world (x, y, theta).
    Returns (value (n,), grad (n, 3) = d/dx, d/dy, d/dtheta, ok (n,) bool)."""
    vol = np.asarray(volume, dtype=np.float64)
    n_yaw, ny, nx = vol.shape
    dth = 2.0 * math.pi / n_yaw
    xyt = np.asarray(xyt, dtype=np.float64).reshape(-1, 3)
    val = np.full(len(xyt), np.nan)
    grad = np.full((len(xyt), 3), np.nan)
    ok = np.zeros(len(xyt), dtype=bool)
    for q, (x, y, th) in enumerate(xyt):
        fx = x / r - 0.5 - I_M                # continuous logical column of the node lattice
        fy = y / r - 0.5 - J_M
        ft = (th + math.pi) / dth             # continuous yaw-bin coordinate
        i0, j0 = math.floor(fx), math.floor(fy)
        tx, ty = fx - i0, fy - j0
        kf = math.floor(ft)
        tt = ft - kf
        k0 = kf % n_yaw                       # SO(2): bins wrap across the seam
        k1 = (k0 + 1) % n_yaw
        if not (0 <= i0 and i0 + 1 < nx and 0 <= j0 and j0 + 1 < ny):
            continue
        v = 0.0
        g = [0.0, 0.0, 0.0]
        for dk, kk, wt in ((0, k0, 1.0 - tt), (1, k1, tt)):
            for dj, wy in ((0, 1.0 - ty), (1, ty)):
                for di, wx in ((0, 1.0 - tx), (1, tx)):
                    c = vol[kk, j0 + dj, i0 + di]
                    v += wx * wy * wt * c
                    g[0] += (1.0 if di else -1.0) * wy * wt * c
                    g[1] += wx * (1.0 if dj else -1.0) * wt * c
                    g[2] += wx * wy * (1.0 if dk else -1.0) * c
        val[q] = v
        grad[q] = (g[0] / r, g[1] / r, g[2] / dth)
        ok[q] = True
    return val, grad, ok
