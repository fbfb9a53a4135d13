"""Seeded synthetic LiDAR frames for the front-end (NEXT-1) — inputs only, none of the method's arithmetic.

A spinning LiDAR (n_beams elevation angles x n_az azimuths) mounted at p_BS on a robot whose true pose
sits on the terrain; each ray is marched through the continuous terrain surface (Hills.surface) and
refined by bisection; the hit is returned in the SENSOR frame with Gaussian range-independent noise
(Sigma_S = sigma_s^2 I).  Rays without a hit within max_range are dropped.  The surface the rays see
is the terrain sampled every 2.5 cm around the robot, bilinear in between.  The method's estimated
pose may differ from the true one by pose noise (Sigma_R, Sigma_B).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def rot_zyx(yaw: float, pitch: float, roll: float) -> np.ndarray:
    cy, sy, cp, sp, cr, sr = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch), math.cos(roll), math.sin(roll)
    Rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1.0]])
    Ry = np.array([[cp, 0, sp], [0, 1.0, 0], [-sp, 0, cp]])
    Rx = np.array([[1.0, 0, 0], [0, cr, -sr], [0, sr, cr]])
    return Rz @ Ry @ Rx


@dataclass
class Frame:
    points_s: np.ndarray      # (n, 3) float32, sensor frame
    R_B: np.ndarray           # estimated pose
    p_B: np.ndarray
    R_BS: np.ndarray
    p_BS: np.ndarray
    Sigma_S: np.ndarray
    Sigma_R: np.ndarray
    Sigma_B: np.ndarray


def scan(terrain, x: float, y: float, yaw: float, seed: int, n_beams: int = 16, n_az: int = 900,
         fov=(-0.45, 0.05), max_range: float = 12.0, step: float = 0.05, sigma_s: float = 0.01,
         mount_h: float = 0.6, body_h: float = 0.3, pose_noise: float = 0.0) -> Frame:
    rng = np.random.default_rng(seed)
    # the surface the rays hit: the terrain sampled on a fine grid around the robot, bilinear in between
    fine = 0.025
    half = max_range + 1.0
    gx0, gy0 = x - half, y - half
    nfg = int(math.ceil(2 * half / fine)) + 2
    xs = gx0 + fine * np.arange(nfg)
    ys = gy0 + fine * np.arange(nfg)
    G = terrain.surface(xs[None, :], ys[:, None])

    def surf(px, py):
        u = np.clip((px - gx0) / fine, 0, nfg - 1.001)
        v = np.clip((py - gy0) / fine, 0, nfg - 1.001)
        i0, j0 = np.floor(u).astype(int), np.floor(v).astype(int)
        a, b = u - i0, v - j0
        return ((1 - a) * (1 - b) * G[j0, i0] + a * (1 - b) * G[j0, i0 + 1] + (1 - a) * b * G[j0 + 1, i0]
                + a * b * G[j0 + 1, i0 + 1])

    zb = float(surf(x, y)) + body_h
    # body attitude from the local terrain slope (finite differences of the true surface)
    e = 0.2
    gx = float(surf(x + e, y) - surf(x - e, y)) / (2 * e)
    gy = float(surf(x, y + e) - surf(x, y - e)) / (2 * e)
    pitch = -math.atan(gx * math.cos(yaw) + gy * math.sin(yaw))
    roll = math.atan(-gx * math.sin(yaw) + gy * math.cos(yaw))
    R_B = rot_zyx(yaw, pitch, roll)
    p_B = np.array([x, y, zb])
    R_BS = np.eye(3)
    p_BS = np.array([0.0, 0.0, mount_h])
    origin = R_B @ p_BS + p_B
    el = np.linspace(fov[0], fov[1], n_beams)
    az = np.linspace(-math.pi, math.pi, n_az, endpoint=False) + rng.uniform(0, 2 * math.pi / n_az)
    E, A = np.meshgrid(el, az, indexing="ij")
    d_s = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], axis=-1).reshape(-1, 3)
    d_w = d_s @ (R_B @ R_BS).T
    n = len(d_w)
    t_prev = np.zeros(n)
    hit = np.full(n, np.nan)
    ts = np.arange(step, max_range + step, step)
    alive = np.ones(n, dtype=bool)
    for t in ts:
        idx = np.nonzero(alive)[0]
        if len(idx) == 0:
            break
        p = origin + d_w[idx] * t
        below = p[:, 2] <= surf(p[:, 0], p[:, 1])
        if below.any():
            b = idx[below]
            lo, hi = np.full(len(b), t - step), np.full(len(b), t)
            for _ in range(30):                          # bisection to ~step / 2^30
                mid = 0.5 * (lo + hi)
                pm = origin + d_w[b] * mid[:, None]
                under = pm[:, 2] <= surf(pm[:, 0], pm[:, 1])
                hi = np.where(under, mid, hi)
                lo = np.where(under, lo, mid)
            hit[b] = 0.5 * (lo + hi)
            alive[b] = False
    ok = np.isfinite(hit)
    pts = d_s[ok] * hit[ok, None] + rng.normal(0.0, sigma_s, size=(ok.sum(), 3))
    R_est, p_est = R_B, p_B
    if pose_noise > 0:
        R_est = R_B @ rot_zyx(*rng.normal(0, pose_noise, 3))
        p_est = p_B + rng.normal(0, pose_noise, 3)
    return Frame(points_s=pts.astype(np.float32), R_B=R_est, p_B=p_est, R_BS=R_BS, p_BS=p_BS,
                 Sigma_S=np.eye(3) * sigma_s ** 2, Sigma_R=np.eye(3) * 1e-6, Sigma_B=np.eye(3) * 1e-5)
