"""Shared setup for the -m gpu tests: build one map through the C ABI and the oracle on the same input."""
from __future__ import annotations

import numpy as np

import oracle
from synth.terrain import CONFIGS, world_heights
from tests.parity import compare


def make_map(nx, ny, r, n_yaw, ex=0.8, ey=0.5, robot=(0.37, 0.61), **kw):
    from paper_2503_02412_b200.se2map import Se2Map
    return Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, ellipse_ex=ex, ellipse_ey=ey,
                  robot_x=robot[0], robot_y=robot[1], **kw)


def oracle_params(nx, ny, r, n_yaw, ex=0.8, ey=0.5):
    return oracle.Params(nx=nx, ny=ny, resolution=r, n_yaw=n_yaw, ex=ex, ey=ey)


def run_config(name=None, cfg=None, known=None, **kw):
    cfg = dict(CONFIGS[name] if name else cfg)
    cfg.update(kw)
    nx, ny, r, n_yaw, ex, ey = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"], cfg["ex"], cfg["ey"]
    x, y = cfg["robot"]
    I_M, J_M = oracle.window_origin(x, y, r, nx, ny)
    h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
    m = make_map(nx, ny, r, n_yaw, ex, ey, robot=(x, y))
    assert m.origin() == (I_M, J_M)
    m.update_elevation(h, known)
    m.assess_se2(0)
    gpu = m.download()
    orc = oracle.assess_all(oracle_params(nx, ny, r, n_yaw, ex, ey), h, known)
    return m, h, gpu, orc, compare(gpu, orc)
