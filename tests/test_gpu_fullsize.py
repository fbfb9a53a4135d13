"""Parity at BASELINE.json's full sizes (high-res 800x800x72 @ 0.05 m, large 2000x2000x72 @ 0.1 m), in
the launch configuration bench.py times (one FULL assess of the whole window), on sampled states the
oracle computes one by one: uniform random states plus a band along the window edges (clipped
footprints) and every yaw bin of a few fixed cells.  Outputs are read through se2m_query, so the
world -> (cell, bin) indexing of the C ABI is exercised at full size too.
"""
import math

import numpy as np
import pytest

import oracle
from synth.terrain import CONFIGS, world_heights
from tests.gpu_common import make_map, oracle_params
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _samples(nx, ny, n_yaw, R, rng, n_uniform=60000, n_edge=20000):
    u = np.stack([rng.integers(0, nx, n_uniform), rng.integers(0, ny, n_uniform),
                  rng.integers(0, n_yaw, n_uniform)], axis=1)
    band = R + 2
    side = rng.integers(0, 4, n_edge)
    a = rng.integers(0, band, n_edge)
    i = np.where(side == 0, a, np.where(side == 1, nx - 1 - a, rng.integers(0, nx, n_edge)))
    j = np.where(side == 2, a, np.where(side == 3, ny - 1 - a, rng.integers(0, ny, n_edge)))
    e = np.stack([i, j, rng.integers(0, n_yaw, n_edge)], axis=1)
    cells = [(0, 0), (nx - 1, ny - 1), (nx // 2, ny // 2), (nx // 3, 2 * ny // 3)]
    f = np.array([(ci, cj, k) for ci, cj in cells for k in range(n_yaw)])
    return np.concatenate([u, e, f]).astype(np.int32)


@pytest.mark.parametrize("name", ["highres", "large"])
def test_fullsize_sampled_parity(name):
    cfg = CONFIGS[name]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    m = make_map(nx, ny, r, n_yaw, robot=cfg["robot"])
    I_M, J_M = m.origin()
    assert (I_M, J_M) == oracle.window_origin(*cfg["robot"], r, nx, ny)
    h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
    m.update_elevation(h)
    m.assess_se2(0)
    R = m.stencil_info(0)[1]
    ijk = _samples(nx, ny, n_yaw, R, np.random.default_rng(17))
    # query at cell centres and exact bin angles (reading R3/R6)
    x = (I_M + ijk[:, 0] + 0.5) * r
    y = (J_M + ijk[:, 1] + 0.5) * r
    th = -math.pi + 2 * math.pi * ijk[:, 2] / n_yaw
    q = m.query(np.stack([x, y, th], axis=1))
    assert q["status"] == 0
    orc = oracle.assess_states(oracle_params(nx, ny, r, n_yaw), h, ijk)
    rep = compare({k: q[k] for k in ("risk", "pitch", "roll", "z", "trav")}, orc)
    print(name, rep)
    assert rep["ok"], rep
    assert rep["normal"] > 0.95 * rep["n"]


@pytest.mark.parametrize("ex,ey,holes", [(1.15, 0.7, 0.0), (1.55, 1.05, 0.0), (1.15, 0.7, 0.03)])
def test_chain_map_big_footprints_sampled_parity(ex, ey, holes):
    """Yaw-chain maps (>= 512^2 cells: period-9 chain, single-cell entries) with footprints of radius 23
    and 31 cells at 0.05 m (kernel tiles R_T = 24 and 32, TY = 16), with and without unknown blobs
    (border / unknown tiles on the chain with validity moments), against the oracle on sampled states."""
    nx, ny, r, n_yaw = 560, 528, 0.05, 72
    terrain = CONFIGS["highres"]["terrain"]
    robot = (-7.31, 4.43)
    m = make_map(nx, ny, r, n_yaw, ex=ex, ey=ey, robot=robot)
    I_M, J_M = m.origin()
    h = world_heights(terrain, I_M, J_M, nx, ny, r)
    known = None
    if holes:
        rng = np.random.default_rng(5)
        known = np.ones((ny, nx), np.uint8)
        nb = int(holes * nx * ny / 49)
        cj, ci = rng.integers(0, ny - 7, nb), rng.integers(0, nx - 7, nb)
        for dj in range(7):
            for di in range(7):
                known[cj + dj, ci + di] = 0
    m.update_elevation(h, known)
    m.assess_se2(0)
    R = m.stencil_info(0)[1]
    assert R >= 22
    ijk = _samples(nx, ny, n_yaw, R, np.random.default_rng(23), n_uniform=12000, n_edge=4000)
    x = (I_M + ijk[:, 0] + 0.5) * r
    y = (J_M + ijk[:, 1] + 0.5) * r
    th = -math.pi + 2 * math.pi * ijk[:, 2] / n_yaw
    q = m.query(np.stack([x, y, th], axis=1))
    orc = oracle.assess_states(oracle_params(nx, ny, r, n_yaw, ex, ey), h, ijk, known=known)
    rep = compare({k: q[k] for k in ("risk", "pitch", "roll", "z", "trav")}, orc)
    print(ex, ey, holes, rep)
    assert rep["ok"], rep


def test_highres_every_state_parity():
    """Every one of the 46.08 M states of the high-res configuration (800 x 800 x 72 @ 0.05 m) in the bench's
    launch configuration (one FULL assess), against the FP64 oracle, one yaw bin at a time (all cells of the
    bin per oracle call)."""
    cfg = CONFIGS["highres"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    m = make_map(nx, ny, r, n_yaw, robot=cfg["robot"])
    I_M, J_M = m.origin()
    h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
    m.update_elevation(h)
    m.assess_se2(0)
    g = m.download()
    m.close()
    P = oracle_params(nx, ny, r, n_yaw)
    jj, ii = np.meshgrid(np.arange(ny, dtype=np.int32), np.arange(nx, dtype=np.int32), indexing="ij")
    tot = None
    for k in range(n_yaw):
        ijk = np.stack([ii.ravel(), jj.ravel(), np.full(nx * ny, k, np.int32)], axis=1)
        orc = oracle.assess_states(P, h, ijk)
        rep = compare({f: g[f][k].ravel() for f in ("risk", "pitch", "roll", "z", "trav")}, orc)
        if tot is None:
            tot = rep
        else:
            for key, v in rep.items():
                if key.startswith("max_"):
                    tot[key] = max(tot[key], v)
                elif key == "ok":
                    tot[key] = tot[key] and v
                elif isinstance(v, int):
                    tot[key] += v
        assert rep["ok"], (k, rep)
    print("highres all states", tot)
    assert tot["n"] == nx * ny * n_yaw and tot["normal"] > 0.95 * tot["n"]
