"""Pins for the trilinear-query oracle.  CPU only."""
import math

import numpy as np
import pytest

from oracle.trilinear import trilinear


def _node_xyt(I_M, J_M, r, n, i, j, k):
    return ((I_M + i + 0.5) * r, (J_M + j + 0.5) * r, -math.pi + 2 * math.pi * k / n)


def test_nodes_and_midpoints():
    rng = np.random.default_rng(1)
    n, ny, nx, r, I_M, J_M = 8, 6, 7, 0.1, -13, 4
    vol = rng.random((n, ny, nx))
    for _ in range(50):
        i, j, k = rng.integers(0, nx - 1), rng.integers(0, ny - 1), rng.integers(0, n)
        v, g, ok = trilinear(vol, I_M, J_M, r, [_node_xyt(I_M, J_M, r, n, i, j, k)])
        assert ok[0] and abs(v[0] - vol[k, j, i]) < 1e-12          # lattice node: stored value
        x, y, th = _node_xyt(I_M, J_M, r, n, i, j, k)
        v, g, ok = trilinear(vol, I_M, J_M, r, [(x, y, th + math.pi / n)])
        assert abs(v[0] - 0.5 * (vol[k, j, i] + vol[(k + 1) % n, j, i])) < 1e-12   # midpoint in theta (cyclic)


def test_affine_reproduction_and_gradient():
    n, ny, nx, r, I_M, J_M = 12, 9, 10, 0.25, 3, -7
    a, b, c, d = 0.7, -1.3, 2.1, 0.4
    kk, jj, ii = np.meshgrid(np.arange(n), np.arange(ny), np.arange(nx), indexing="ij")
    x = (I_M + ii + 0.5) * r
    y = (J_M + jj + 0.5) * r
    th = -math.pi + 2 * math.pi * kk / n
    vol = a + b * x + c * y + d * th
    rng = np.random.default_rng(2)
    q = np.stack([rng.uniform((I_M + 0.5) * r, (I_M + nx - 0.5) * r, 500),
                  rng.uniform((J_M + 0.5) * r, (J_M + ny - 0.5) * r, 500),
                  rng.uniform(-math.pi, math.pi - 2 * math.pi / n, 500)], axis=1)   # not across the seam
    v, g, ok = trilinear(vol, I_M, J_M, r, q)
    assert ok.all()
    assert np.max(np.abs(v - (a + b * q[:, 0] + c * q[:, 1] + d * q[:, 2]))) < 1e-12
    assert np.max(np.abs(g - np.array([b, c, d]))) < 1e-11


def test_seam_matches_unwrapped_duplicate_layer():
    """Across +-pi the cyclic interpolation equals interpolation on a volume with layer n = layer 0."""
    rng = np.random.default_rng(3)
    n, ny, nx, r, I_M, J_M = 6, 5, 5, 0.1, 0, 0
    vol = rng.random((n, ny, nx))
    ext = np.concatenate([vol, vol[:1]], axis=0)               # duplicate layer, unwrapped theta
    dth = 2 * math.pi / n
    for _ in range(200):
        x, y = rng.uniform(0.05, 0.45), rng.uniform(0.05, 0.45)
        t = rng.uniform(0, 1)
        th = math.pi - dth + t * dth                               # between the last bin and the seam
        v, g, ok = trilinear(vol, I_M, J_M, r, [(x, y, th)])
        # independent unwrapped evaluation: bins n-1 and n (= 0) with weight t
        fx, fy = x / r - 0.5, y / r - 0.5
        i0, j0 = int(math.floor(fx)), int(math.floor(fy))
        tx, ty = fx - i0, fy - j0
        plane = lambda L: ((1 - tx) * (1 - ty) * ext[L, j0, i0] + tx * (1 - ty) * ext[L, j0, i0 + 1]
                           + (1 - tx) * ty * ext[L, j0 + 1, i0] + tx * ty * ext[L, j0 + 1, i0 + 1])
        assert abs(v[0] - ((1 - t) * plane(n - 1) + t * plane(n))) < 1e-12
        assert abs(g[0][2] - (plane(n) - plane(n - 1)) / dth) < 1e-9
        # theta and theta - 2 pi are the same state
        v2, _, _ = trilinear(vol, I_M, J_M, r, [(x, y, th - 2 * math.pi)])
        assert abs(v2[0] - v[0]) < 1e-12


def test_gradient_is_derivative_of_interpolant():
    rng = np.random.default_rng(4)
    n, ny, nx, r = 8, 6, 6, 0.1
    vol = rng.random((n, ny, nx))
    for _ in range(100):
        p0 = np.array([rng.uniform(0.07, 0.53), rng.uniform(0.07, 0.53), rng.uniform(-3.1, 3.1)])
        v, g, ok = trilinear(vol, 0, 0, r, [p0])
        for ax, h in ((0, 1e-7), (1, 1e-7), (2, 1e-7)):
            p1 = p0.copy()
            p1[ax] += h
            v1, _, ok1 = trilinear(vol, 0, 0, r, [p1])
            # stay inside the same interpolation cell (piecewise-linear interpolant)
            if ok1[0]:
                fd = (v1[0] - v[0]) / h
                assert abs(fd - g[0][ax]) < 1e-5 * max(1.0, abs(g[0][ax]))


def test_out_of_range():
    vol = np.zeros((4, 3, 3))
    _, _, ok = trilinear(vol, 0, 0, 0.1, [(0.01, 0.1, 0.0), (0.1, 0.1, 0.0), (0.26, 0.1, 0.0)])
    assert list(ok) == [False, True, False]
