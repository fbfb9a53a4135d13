"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no footprint, no covariance, no
eigen-solve, no risk).  It only produces elevation maps and robot paths, the inputs
both sides consume.  Every generator is a pure function of (seed, world cell), is
evaluated in float64 at world cell centres and rounded ONCE to float32, so the oracle
and the GPU read the same array.

Stand-ins for the paper's EPFL-generator terrains (§VII.A), which are
not available:

* ``plane_sine``: h = h0 + tan(alpha)*(x cos(beta) + y sin(beta)) + A sin(2 pi x/lx) cos(2 pi y/ly)
* ``hills``:      h = h0 + sum_k a_k sin(2 pi/lambda_k * (x cos psi_k + y sin psi_k) + phi_k) + eps(I, J)
  with lambda_k = exp(U[ln 1.5, ln 12]) m, a_k = slope_rms*lambda_k/(2 pi sqrt(K/2)) (so the RMS
  gradient is slope_rms) and eps(I, J) = sigma*N(0,1) from a splitmix64 hash of (seed, I, J),
  i.e. a pure function of the WORLD cell, so the rolling-window stream can generate newly
  exposed strips on the fly.

World cell I covers [I*r, (I+1)*r) and its centre is (I + 1/2)*r (reading R6).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _cell_hash(seed: int, I: np.ndarray, J: np.ndarray, stream: int) -> np.ndarray:
    """Counter-based hash of (seed, I, J, stream) -> uint64."""
    with np.errstate(over="ignore"):
        key = np.uint64(seed & 0xFFFFFFFF) * np.uint64(0x100000001B3) + np.uint64(stream)
        a = I.astype(np.int64).astype(np.uint64)
        b = J.astype(np.int64).astype(np.uint64)
        h = _splitmix64(key ^ _splitmix64(a * np.uint64(0xD6E8FEB86659FD93)))
        return _splitmix64(h ^ _splitmix64(b * np.uint64(0xA0761D6478BD642F) + np.uint64(1)))


def cell_normal_noise(seed: int, I: np.ndarray, J: np.ndarray) -> np.ndarray:
    """N(0,1) per world cell by Box-Muller over two independent uniform hashes."""
    u1 = (_cell_hash(seed, I, J, 1) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    u2 = (_cell_hash(seed, I, J, 2) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    u1 = np.maximum(u1, 1e-300)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


@dataclass(frozen=True)
class PlaneSine:
    alpha: float = 0.25
    beta: float = 0.6
    h0: float = 50.0
    A: float = 0.05
    lx: float = 0.7
    ly: float = 0.9

    def height64(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        t = math.tan(self.alpha)
        return (self.h0 + t * (x * math.cos(self.beta) + y * math.sin(self.beta))
                + self.A * np.sin(2.0 * math.pi * x / self.lx) * np.cos(2.0 * math.pi * y / self.ly))


@dataclass(frozen=True)
class Plane:
    """h = h0 + gx*x + gy*y exactly (choose dyadic gx, gy, h0, r for exact float32 values)."""
    gx: float = 0.0
    gy: float = 0.0
    h0: float = 0.0

    def height64(self, x, y):
        return self.h0 + self.gx * x + self.gy * y


@dataclass(frozen=True)
class Hills:
    seed: int = 1
    K: int = 24
    slope_rms: float = 0.5
    h0: float = 100.0
    sigma: float = 0.01
    lam_min: float = 1.5
    lam_max: float = 12.0
    rock_density: float = 0.2    # probability of one rock per 1 m x 1 m world block
    rock_block: float = 1.0

    def components(self):
        rng = np.random.Generator(np.random.PCG64(self.seed))
        lam = np.exp(rng.uniform(math.log(self.lam_min), math.log(self.lam_max), self.K))
        psi = rng.uniform(0.0, 2.0 * math.pi, self.K)
        phi = rng.uniform(0.0, 2.0 * math.pi, self.K)
        amp = self.slope_rms * lam / (2.0 * math.pi * math.sqrt(self.K / 2.0))
        return lam, psi, phi, amp

    def height64(self, x: np.ndarray, y: np.ndarray, I: np.ndarray, J: np.ndarray) -> np.ndarray:
        lam, psi, phi, amp = self.components()
        h = np.full(np.broadcast(x, y).shape, self.h0, dtype=np.float64)
        for k in range(self.K):
            h += amp[k] * np.sin(2.0 * math.pi / lam[k] * (x * math.cos(psi[k]) + y * math.sin(psi[k])) + phi[k])
        if self.sigma:
            h += self.sigma * cell_normal_noise(self.seed, I, J)
        if self.rock_density > 0:
            h += self.rocks(x, y)
        return h

    def surface(self, x, y):
        """The continuous terrain surface (hills + rocks, no per-cell noise): what a LiDAR sees."""
        lam, psi, phi, amp = self.components()
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        h = np.full(np.broadcast(x, y).shape, self.h0, dtype=np.float64)
        for k in range(self.K):
            h += amp[k] * np.sin(2.0 * math.pi / lam[k] * (x * math.cos(psi[k]) + y * math.sin(psi[k])) + phi[k])
        if self.rock_density > 0:
            h += self.rocks(x, y)
        return h

    def rocks(self, x, y):
        """Sparse Gaussian bumps ('rocks'): at most one per rock_block-sized world block, placed and
        sized by a hash of (seed, block) so that they are a pure function of world position.
        Height U[0.2, 0.6] m, radius U[0.1, 0.3] m; they make the curvature term kappa matter."""
        B = self.rock_block
        x = np.broadcast_to(x, np.broadcast(x, y).shape)
        y = np.broadcast_to(y, x.shape)
        bi0 = np.floor(x / B).astype(np.int64)
        bj0 = np.floor(y / B).astype(np.int64)
        out = np.zeros(x.shape, dtype=np.float64)
        to_u = lambda v: (v >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        for oj in (-1, 0, 1):
            for oi in (-1, 0, 1):
                bi, bj = bi0 + oi, bj0 + oj
                present = to_u(_cell_hash(self.seed + 7919, bi, bj, 3)) < self.rock_density
                cx = (bi + to_u(_cell_hash(self.seed + 7919, bi, bj, 4))) * B
                cy = (bj + to_u(_cell_hash(self.seed + 7919, bi, bj, 5))) * B
                ht = 0.2 + 0.4 * to_u(_cell_hash(self.seed + 7919, bi, bj, 6))
                rad = 0.1 + 0.2 * to_u(_cell_hash(self.seed + 7919, bi, bj, 7))
                d2 = (x - cx) ** 2 + (y - cy) ** 2
                out += np.where(present, ht * np.exp(-d2 / (2.0 * rad * rad)), 0.0)
        return out


def world_heights(terrain, I0: int, J0: int, nx: int, ny: int, r: float) -> np.ndarray:
    """float32 heights of world cells [I0, I0+nx) x [J0, J0+ny), array shape (ny, nx), x fastest."""
    I = np.arange(I0, I0 + nx, dtype=np.int64)[None, :]
    J = np.arange(J0, J0 + ny, dtype=np.int64)[:, None]
    x = (I.astype(np.float64) + 0.5) * r
    y = (J.astype(np.float64) + 0.5) * r
    if isinstance(terrain, Hills):
        h = terrain.height64(x, y, np.broadcast_to(I, (ny, nx)), np.broadcast_to(J, (ny, nx)))
    else:
        h = terrain.height64(x, y)
    h = np.broadcast_to(h, (ny, nx))
    return np.ascontiguousarray(h.astype(np.float32))


def robot_path(seed: int, n_steps: int, r: float, x0: float, y0: float,
               psi_sigma: float = 0.1, step_min: float = 0.05, step_max: float = 0.35):
    """Stream path (SURVEY.md §8(d) 'stream'): heading random walk, U[step_min, step_max] steps.

    Positions within 1e-6*r of a cell boundary are re-drawn so that floor(x/r) is never a
    rounding coin-flip (reading R7).  Returns an (n_steps+1, 2) float64 array.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    pts = [(x0, y0)]
    x, y, psi = x0, y0, rng.uniform(0, 2 * math.pi)

    def near_boundary(v):
        q = v / r
        return abs(q - round(q)) < 1e-6

    for _ in range(n_steps):
        while True:
            npsi = psi + rng.normal(0.0, psi_sigma)
            d = rng.uniform(step_min, step_max)
            nx_, ny_ = x + d * math.cos(npsi), y + d * math.sin(npsi)
            if not (near_boundary(nx_) or near_boundary(ny_)):
                break
        x, y, psi = nx_, ny_, npsi
        pts.append((x, y))
    return np.array(pts, dtype=np.float64)


# ---- the benchmark configurations of BASELINE.json ----------------------
CONFIGS = {
    "tiny": dict(nx=20, ny=20, r=0.1, n_yaw=8, ex=0.8, ey=0.5, robot=(1.03, 2.07),
                 terrain=PlaneSine(alpha=0.25, beta=0.6, h0=50.0, A=0.05, lx=0.7, ly=0.9)),
    "tiny_small_fp": dict(nx=20, ny=20, r=0.1, n_yaw=8, ex=0.3, ey=0.2, robot=(1.03, 2.07),
                          terrain=PlaneSine(alpha=0.25, beta=0.6, h0=50.0, A=0.05, lx=0.7, ly=0.9)),
    "paper": dict(nx=100, ny=100, r=0.1, n_yaw=36, ex=0.8, ey=0.5, robot=(0.37, 0.61),
                  terrain=Hills(seed=1)),
    "stream": dict(nx=100, ny=100, r=0.1, n_yaw=36, ex=0.8, ey=0.5, robot=(0.37, 0.61),
                   terrain=Hills(seed=2), path_seed=3, n_steps=1000),
    "highres": dict(nx=800, ny=800, r=0.05, n_yaw=72, ex=0.8, ey=0.5, robot=(0.37, 0.61),
                    terrain=Hills(seed=4)),
    "large": dict(nx=2000, ny=2000, r=0.1, n_yaw=72, ex=0.8, ey=0.5, robot=(0.37, 0.61),
                  terrain=Hills(seed=5)),
}

DEFAULT_RISK = dict(w=(0.4, 0.3, 0.3), kappa_max=0.1, phi_x_max=0.52, phi_y_max=0.52)
