#!/usr/bin/env python
"""Small end-to-end cases of the library for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py CASE

Each case drives the C ABI through the ctypes binding on a map small enough that the sanitizer's
instrumentation finishes in seconds, and covers one group of kernels:

  tiny      init, update_elevation, assess FULL, shift_window, INCREMENTAL, query, query_async, downloads
  chain     544 x 520 x 36 (yaw chain, TMA halo loads, vertical-window-edge kernel <8, 1> on its stream)
  highres   160 x 160 x 16 @ 0.05 m (R_T = 16 tiles), FULL + INCREMENTAL
  holes     paper-like window with 20 % unknown cells (general path, direct FP64 states)
  step      se2m_step (H1 + H2 + H9 in one call) over 30 rolling-window steps
  halo      row-band shards (G = 2) with se2m_halo_pack / _unpack handed over by device copies
  next      SDF, trilinear, inpainting and the LiDAR front-end (NEXT-1..4)
  all       every case above in one process
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth.terrain import CONFIGS, world_heights  # noqa: E402


def _map(S, nx, ny, r, n_yaw, robot=(0.37, 0.61), **kw):
    return S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=robot[0], robot_y=robot[1], **kw)


def case_tiny(S):
    c = CONFIGS["tiny"]
    m = _map(S, c["nx"], c["ny"], c["r"], c["n_yaw"], c["robot"], ellipse_ex=c["ex"], ellipse_ey=c["ey"])
    I, J = m.origin()
    m.update_elevation(world_heights(c["terrain"], I, J, c["nx"], c["ny"], c["r"]))
    m.assess_se2(0)
    di, dj = m.shift_window(c["robot"][0] + 0.31, c["robot"][1] - 0.2)
    I, J = m.origin()
    m.update_elevation(world_heights(c["terrain"], I, J, c["nx"], c["ny"], c["r"]))
    m.assess_se2(1)
    q = np.array([[(I + 3.5) * c["r"], (J + 4.5) * c["r"], 0.3], [1e6, 0, 0]])
    m.query(q)
    import torch
    xyt = torch.from_numpy(q).pin_memory()
    out = torch.empty((5, 2), dtype=torch.float32).pin_memory()
    m.query_async(xyt, out)
    m.synchronize()
    m.download()
    m.download_compact()
    m.download_compact_rep()
    m.synchronize()
    m.close()


def case_chain(S):
    nx, ny = 544, 520
    m = _map(S, nx, ny, 0.1, 36, robot=(3.37, -2.61))
    I, J = m.origin()
    m.update_elevation(world_heights(CONFIGS["large"]["terrain"], I, J, nx, ny, 0.1))
    m.assess_se2(0)
    m.shift_window(3.37 + 0.45, -2.61 + 0.33)
    I, J = m.origin()
    m.update_elevation(world_heights(CONFIGS["large"]["terrain"], I, J, nx, ny, 0.1))
    m.assess_se2(1)
    m.download(planes=("risk", "trav"))
    m.close()


def case_highres(S):
    nx = ny = 160
    m = _map(S, nx, ny, 0.05, 16, robot=(1.03, 2.07))
    I, J = m.origin()
    m.update_elevation(world_heights(CONFIGS["highres"]["terrain"], I, J, nx, ny, 0.05))
    m.assess_se2(0)
    m.shift_window(1.03 + 0.2, 2.07 + 0.1)
    I, J = m.origin()
    m.update_elevation(world_heights(CONFIGS["highres"]["terrain"], I, J, nx, ny, 0.05))
    m.assess_se2(1)
    m.download(planes=("risk",))
    m.close()


def case_holes(S):
    c = CONFIGS["paper"]
    m = _map(S, c["nx"], c["ny"], c["r"], 12, c["robot"])
    I, J = m.origin()
    h = world_heights(c["terrain"], I, J, c["nx"], c["ny"], c["r"])
    known = (np.random.default_rng(3).random(h.shape) > 0.2).astype(np.uint8)
    m.update_elevation(h, known)
    m.assess_se2(0)
    m.download(planes=("risk", "pitch"))
    m.close()


def case_step(S):
    import torch
    from synth.terrain import robot_path
    c = CONFIGS["stream"]
    nx, ny, r = c["nx"], c["ny"], c["r"]
    m = _map(S, nx, ny, r, c["n_yaw"], c["robot"])
    path = robot_path(c["path_seed"], 30, r, *c["robot"])
    I0 = int(math.floor(path[:, 0].min() / r)) - nx // 2 - 2
    J0 = int(math.floor(path[:, 1].min() / r)) - ny // 2 - 2
    W = int(math.ceil((path[:, 0].max() - path[:, 0].min()) / r)) + nx + 6
    H = int(math.ceil((path[:, 1].max() - path[:, 1].min()) / r)) + ny + 6
    wh = torch.from_numpy(world_heights(c["terrain"], I0, J0, W, H, r)).cuda()
    I, J = m.origin()
    m.update_elevation(world_heights(c["terrain"], I, J, nx, ny, r))
    m.assess_se2(0)
    for t in range(1, len(path)):
        m.step(*path[t], wh, I0, J0)
    m.synchronize()
    m.close()


def case_halo(S):
    import torch
    nx, ny, G = 256, 200, 2
    maps = [_map(S, nx, ny, 0.1, 12, robot=(1.1, 0.4), shard_mode=2, rank=g, world_size=G) for g in range(G)]
    I, J = maps[0].origin()
    h = world_heights(CONFIGS["large"]["terrain"], I, J, nx, ny, 0.1)
    for m in maps:
        for j in m.owned_rows():
            m.update_elevation(np.ascontiguousarray(h[j:j + 1]), j0=int(j))
    cap, rows = maps[0].halo_size()
    lo, hi = [], []
    for m in maps:
        a = torch.empty((cap, rows, nx), dtype=torch.float32, device="cuda")
        b = torch.empty_like(a)
        m.halo_pack(-1, a)
        m.halo_pack(+1, b)
        m.synchronize()
        lo.append(a)
        hi.append(b)
    for g, m in enumerate(maps):
        m.halo_unpack(lo[(g + 1) % G], +1)
        m.halo_unpack(hi[(g - 1) % G], -1)
        m.assess_se2(0)
        m.download_compact_rep()
        m.synchronize()
    for m in maps:
        m.close()


def case_next(S):
    c = CONFIGS["paper"]
    m = _map(S, c["nx"], c["ny"], c["r"], c["n_yaw"], c["robot"])
    I, J = m.origin()
    h = world_heights(c["terrain"], I, J, c["nx"], c["ny"], c["r"])
    m.update_elevation(h)
    m.assess_se2(0)
    m.compute_sdf(1.0)
    m.download_sdf()
    rng = np.random.default_rng(0)
    r = c["r"]
    q = np.stack([rng.uniform((I + 1) * r, (I + c["nx"] - 1) * r, 512), rng.uniform((J + 1) * r, (J + c["ny"] - 1) * r, 512),
                  rng.uniform(-math.pi, math.pi, 512)], 1)
    m.query_trilinear(q, 0)
    m.query_trilinear(q, 1)
    known = (rng.random(h.shape) > 0.6).astype(np.uint8)
    m.update_elevation(h, known)
    m.inpaint()
    m.download_inpainted()
    S.sdf_from_mask((rng.random((2, 40, 50)) > 0.8).astype(np.uint8), 0.1, 0.5)
    from synth.lidar import scan
    from synth.terrain import Hills
    fr = scan(Hills(seed=31), 0.37, 0.61, 0.3, seed=5, n_az=200)
    pose = S.Pose.from_arrays(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S, fr.Sigma_R, fr.Sigma_B)
    m2 = _map(S, 180, 180, 0.1, 30, robot=(0.37, 0.61), inpaint=1)
    m2.integrate_scan(fr.points_s, pose)
    m2.assess_se2(0)
    m2.synchronize()
    m2.close()
    m.close()


CASES = {"tiny": case_tiny, "chain": case_chain, "highres": case_highres, "holes": case_holes,
         "step": case_step, "halo": case_halo, "next": case_next}


def main():
    from paper_2503_02412_b200 import se2map as S
    names = sys.argv[1:] or ["all"]
    if names == ["all"]:
        names = list(CASES)
    for n in names:
        CASES[n](S)
        print("case", n, "done", flush=True)


if __name__ == "__main__":
    main()
