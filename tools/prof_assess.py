#!/usr/bin/env python
"""Time (or, under ncu, just launch) one configuration's FULL assess through the C ABI.

    python tools/prof_assess.py --config large [--holes 0.02] [--reps 10]

--holes f: that fraction of cells is unknown, in 3x3 blobs at random places (LiDAR shadows), which
sends most tiles down the general (border / unknown) path.  Prints ms per FULL assess (host wall clock
around assess + synchronize; the kernel dominates at these sizes).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from synth.terrain import CONFIGS, world_heights  # noqa: E402


def _segments(m):
    try:
        return m.chain_segments()
    except Exception:  # an A/B build from before se2m_chain_segments
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large", choices=sorted(CONFIGS))
    ap.add_argument("--holes", type=float, default=0.0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sdf", type=float, default=0.0, help="also time compute_sdf(d_max) after the assess")
    ap.add_argument("--segments", type=int, default=0, help="params.chain_segments (0 = auto)")
    ap.add_argument("--scan", action="store_true",
                    help="the bench's paper_pipeline map instead: 180x180x30 built from 4 LiDAR frames")
    a = ap.parse_args()
    from paper_2503_02412_b200.se2map import Se2Map

    if a.scan:
        return scan_map(a, Se2Map)
    c = CONFIGS[a.config]
    nx, ny, r = c["nx"], c["ny"], c["r"]
    x, y = c["robot"]
    m = Se2Map(nx=nx, ny=ny, n_yaw=c["n_yaw"], resolution=r, ellipse_ex=c["ex"], ellipse_ey=c["ey"],
               robot_x=x, robot_y=y, chain_segments=a.segments)
    I_M, J_M = m.origin()  # the library's Eq. 4 window origin
    h = world_heights(c["terrain"], I_M, J_M, nx, ny, r)
    known = None
    if a.holes > 0:
        rng = np.random.default_rng(0)
        known = np.ones((ny, nx), np.uint8)
        nb = int(a.holes * nx * ny / 9)
        ci, cj = rng.integers(1, nx - 1, nb), rng.integers(1, ny - 1, nb)
        for di in (-1, 0, 1):
            for dj in (-1, 0, 1):
                known[cj + dj, ci + di] = 0
    m.update_elevation(h, known)
    m.assess_se2(0)
    m.synchronize()
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        m.assess_se2(0)
        m.synchronize()
        ts.append(time.perf_counter() - t)
    res = dict(config=a.config, holes=a.holes, segments=_segments(m), unknown_frac=0.0 if known is None else float(1 - known.mean()),
               ms_median=1e3 * float(np.median(ts)), ms_min=1e3 * float(np.min(ts)))
    if a.sdf > 0:
        m.compute_sdf(a.sdf)
        m.synchronize()
        ts = []
        for _ in range(a.reps):
            t = time.perf_counter()
            m.compute_sdf(a.sdf)
            m.synchronize()
            ts.append(time.perf_counter() - t)
        res["sdf_ms_median"] = 1e3 * float(np.median(ts))
    print(json.dumps(res))


def scan_map(a, Se2Map):
    from paper_2503_02412_b200 import se2map as S
    from synth.lidar import scan
    from synth.terrain import Hills
    terrain = Hills(seed=31)
    path = [(0.37 + 0.15 * t, 0.61 + 0.05 * t, 0.3 + 0.02 * t) for t in range(4)]
    m = Se2Map(nx=180, ny=180, n_yaw=30, resolution=0.1, robot_x=path[0][0], robot_y=path[0][1])
    for t, (x, y, yaw) in enumerate(path):
        fr = scan(terrain, x, y, yaw, seed=500 + t, n_az=1800)
        m.shift_window(x, y)
        m.integrate_scan(fr.points_s, S.Pose.from_arrays(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S,
                                                         fr.Sigma_R, fr.Sigma_B))
    h, _ = m.download_elevation()
    m.assess_se2(0)
    m.synchronize()
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        m.assess_se2(0)
        m.synchronize()
        ts.append(time.perf_counter() - t)
    print(json.dumps(dict(config="scan180", unknown_frac=float(np.isnan(h).mean()),
                          ms_median=1e3 * float(np.median(ts)), ms_min=1e3 * float(np.min(ts)))))


if __name__ == "__main__":
    main()
