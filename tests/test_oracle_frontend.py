"""Pins for the front-end oracle (NEXT-1).  CPU only."""
import math

import numpy as np
import pytest

import oracle
from oracle.frontend import FrontendParams, Pose, integrate_scan, point_measurement
from synth.lidar import rot_zyx


def _skew(v):
    return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0.0]])


def _expm_so3(w):
    th = np.linalg.norm(w)
    if th < 1e-12:
        return np.eye(3) + _skew(w)
    K = _skew(w / th)
    return np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * K @ K


def test_variance_worked_examples():
    """identity rotations, Sigma_S = s^2 I -> s^2; Sigma_B = diag(a, b, c) only -> c."""
    pose = Pose(R_B=np.eye(3), p_B=np.zeros(3), Sigma_S=np.eye(3) * 0.04)
    assert point_measurement([1.0, 2.0, -0.5], pose)[4] == pytest.approx(0.04, abs=1e-18)
    pose = Pose(R_B=np.eye(3), p_B=np.zeros(3), Sigma_B=np.diag([0.1, 0.2, 0.3]))
    assert point_measurement([1.0, 2.0, -0.5], pose)[4] == pytest.approx(0.3, abs=1e-16)


def test_variance_matches_monte_carlo():
    """sigma^2 of PAPER.md:120 vs the empirical variance of z_l under perturbations of the
    sensor point, the attitude (right perturbation on SO(3)) and the position (first-order agreement)."""
    rng = np.random.default_rng(0)
    for trial in range(3):
        R_B = rot_zyx(*rng.uniform(-0.4, 0.4, 3))
        R_BS = rot_zyx(*rng.uniform(-0.2, 0.2, 3))
        p_B, p_BS = rng.normal(0, 1, 3), np.array([0.1, -0.05, 0.6])
        ps = rng.uniform(-4, 4, 3)
        A = rng.normal(size=(3, 3)) * 0.01
        S_S, S_R, S_B = A @ A.T + 1e-5 * np.eye(3), np.diag([2e-5, 1e-5, 3e-5]), np.diag([1e-4, 2e-4, 5e-5])
        pose = Pose(R_B=R_B, p_B=p_B, R_BS=R_BS, p_BS=p_BS, Sigma_S=S_S, Sigma_R=S_R, Sigma_B=S_B)
        s2 = point_measurement(ps, pose)[4]
        n = 100000
        dps = rng.multivariate_normal(np.zeros(3), S_S, n)
        dth = rng.multivariate_normal(np.zeros(3), S_R, n)
        dpb = rng.multivariate_normal(np.zeros(3), S_B, n)
        z = np.empty(n)
        for t in range(n):
            Rt = R_B @ _expm_so3(dth[t])
            z[t] = (Rt @ (R_BS @ (ps + dps[t]) + p_BS) + p_B + dpb[t])[2]
        assert abs(z.var() - s2) < 0.05 * s2, (trial, z.var(), s2)


def _window(nx=12, ny=10, r=0.1):
    w = oracle.Window(nx, ny, r, 0.55, 0.55)
    return w, w.var


def _point_at(w, i, j, z, pose_z=0.0):
    """Sensor-frame point landing in window cell (i, j) at height z for an identity pose at p_B = (0, 0, pose_z)."""
    x = (w.I_M + i + 0.5) * w.r
    y = (w.J_M + j + 0.5) * w.r
    return [x, y, z - pose_z]


def test_kf_worked_examples():
    """equal-variance fusion; unknown -> initialise; gate failure -> higher wins."""
    P = FrontendParams(z_min=-10, z_max=10)
    w, var = _window()
    w.known[4, 5] = 1; w.heights[4, 5] = 0.0; var[4, 5] = 1.0
    pose = Pose(R_B=np.eye(3), p_B=np.zeros(3), Sigma_S=np.eye(3))            # sigma_m^2 = 1
    integrate_scan(w, [_point_at(w, 5, 4, 1.0)], pose, P)
    assert (w.heights[4, 5], var[4, 5]) == (np.float32(0.5), np.float32(0.5))
    w, var = _window()
    pose = Pose(R_B=np.eye(3), p_B=np.zeros(3), Sigma_S=np.eye(3) * 0.04)
    integrate_scan(w, [_point_at(w, 2, 3, 2.0)], pose, P)
    assert (w.known[3, 2], w.heights[3, 2], var[3, 2]) == (1, np.float32(2.0), np.float32(0.04))
    w, var = _window()
    w.known[4, 5] = 1; w.heights[4, 5] = 0.0; var[4, 5] = 1e-4
    pose = Pose(R_B=np.eye(3), p_B=np.zeros(3), Sigma_S=np.eye(3) * 1e-4)
    integrate_scan(w, [_point_at(w, 5, 4, 0.5)], pose, P)                 # d = 35.36 > 2, higher
    assert (w.heights[4, 5], var[4, 5]) == (np.float32(0.5), np.float32(1e-4))
    integrate_scan(w, [_point_at(w, 5, 4, -0.5)], pose, P)                # gate fails, lower: discarded
    assert (w.heights[4, 5], var[4, 5]) == (np.float32(0.5), np.float32(1e-4))


def test_kf_properties():
    """Ungated fusion: order-insensitive (to float32 storage precision), variance non-increasing."""
    rng = np.random.default_rng(3)
    P = FrontendParams(z_min=-10, z_max=10, gate=1e9)
    zs = rng.normal(1.0, 0.01, 20)
    res = []
    for order in (np.arange(20), rng.permutation(20)):
        w, var = _window()
        w.known[4, 5] = 1; w.heights[4, 5] = 1.0; var[4, 5] = 1e-3
        pose = Pose(R_B=np.eye(3), p_B=np.zeros(3), Sigma_S=np.eye(3) * 1e-4)
        prev = var[4, 5]
        for t in order:
            integrate_scan(w, [_point_at(w, 5, 4, zs[t])], pose, P)
            assert var[4, 5] <= prev
            prev = var[4, 5]
        res.append((float(w.heights[4, 5]), float(var[4, 5])))
    assert abs(res[0][0] - res[1][0]) < 1e-6 and abs(res[0][1] - res[1][1]) < 1e-6 * res[0][1]
    # the float64 information form: 1/var = 1/1e-3 + 20/1e-4
    assert res[0][1] == pytest.approx(1.0 / (1e3 + 20 * 1e4), rel=1e-5)


def test_raycast_worked_examples_and_filters():
    """a ghost cell above the ray is reset, a cell below every ray is untouched;
    points outside the window / the height band are not used."""
    P = FrontendParams(z_min=-2.0, z_max=2.0, ray_eps=0.05)
    w, var = _window(nx=30, ny=10)
    w.known[:] = 1; w.heights[:] = 0.0; var[:] = 1e-2
    w.heights[5, 10] = 1.0                       # ghost on the ray
    w.heights[5, 12] = 0.15                      # below the ray (ray at ~0.2 m there)
    pose = Pose(R_B=np.eye(3), p_B=np.array([(w.I_M + 2.5) * 0.1, (w.J_M + 5.5) * 0.1, 0.3]),
                Sigma_S=np.eye(3) * 1e-4)
    # ray from (cell 2, z 0.3) to (cell 25, z 0.0) along the row j = 5
    pt = np.array([(w.I_M + 25.5) * 0.1, (w.J_M + 5.5) * 0.1, 0.0]) - pose.p_B
    far = np.array([100.0, 0.0, 0.0])
    high = np.array([0.2, 0.0, 5.0])
    status, n_reset = integrate_scan(w, [pt, far, high], pose, P)
    assert list(status) == [0, 1, 2]
    assert w.known[5, 10] == 0 and w.known[5, 12] == 1 and n_reset == 1
    assert w.known[5, 25] == 1 and w.heights[5, 25] == np.float32(0.0)


def test_raycast_cells_match_dense_sampling():
    """The traversed-cell set of the slab method equals dense sampling of the segment (cells only
    grazed within 1e-6 of a corner excluded), on random rays."""
    from oracle.frontend import _cell_interval
    rng = np.random.default_rng(5)
    r = 0.1
    for _ in range(30):
        s = rng.uniform(-1, 1, 2)
        e = s + rng.uniform(-2, 2, 2)
        d = e - s
        exact = set()
        for I in range(math.floor(min(s[0], e[0]) / r) - 1, math.floor(max(s[0], e[0]) / r) + 2):
            for J in range(math.floor(min(s[1], e[1]) / r) - 1, math.floor(max(s[1], e[1]) / r) + 2):
                if _cell_interval(s[0], s[1], d[0], d[1], I * r, (I + 1) * r, J * r, (J + 1) * r) is not None:
                    exact.add((I, J))
        t = np.linspace(1e-9, 1 - 1e-9, 200001)
        pts = s[None, :] + t[:, None] * d[None, :]
        dense = set(map(tuple, np.floor(pts / r).astype(int)))
        for c in exact ^ dense:
            cx, cy = np.array(c) * r
            corners = np.array([[cx, cy], [cx + r, cy], [cx, cy + r], [cx + r, cy + r]])
            dist = np.abs(np.cross(d, corners - s)) / np.linalg.norm(d)
            assert dist.min() < 1e-5, (c, dist.min())
