#!/usr/bin/env python
"""Per-CTA latency breakdown of the assess kernels (library built with SE2M_PHASES: tools/build_phases.sh).

    SE2M_LIB=abx/libse2map_phases.so python tools/phase_report.py [--config paper|stream|large|highres]

Runs one FULL assess (paper / large / highres) or 50 rolling-window steps (stream, se2m_step) and prints, per
kernel mode, the median / max duration of each phase (halo, tile plane, prefix + tables, states, flush) over
warps, the span of the launch, and the slowest CTAs with their tile flags (fast, pin / pfast pair masks).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from synth.terrain import CONFIGS, robot_path, world_heights  # noqa: E402


def summarize(rec, label):
    out = {"label": label, "warp_records": int(len(rec))}
    if not len(rec):
        return out
    t = rec["t"].astype(np.int64)
    t0 = t[:, 0].min()
    for mode in sorted(set(rec["mode"].tolist())):
        sel = rec["mode"] == mode
        tm = t[sel]
        ph = np.diff(tm, axis=1)  # [warps, 5]
        names = ["halo", "plane", "prefix_tables", "states", "flush"]
        d = {n: {"median_us": float(np.median(ph[:, i]) / 1e3), "max_us": float(ph[:, i].max() / 1e3)}
             for i, n in enumerate(names)}
        d["span_us"] = float((tm[:, 5].max() - tm[:, 0].min()) / 1e3)
        d["warp_total_median_us"] = float(np.median(tm[:, 5] - tm[:, 0]) / 1e3)
        d["warp_total_max_us"] = float((tm[:, 5] - tm[:, 0]).max() / 1e3)
        key = rec["bx"][sel].astype(np.int64) * 100000 + rec["by"][sel]
        ctas = {}
        for k, a, b, f, st in zip(key, tm[:, 0], tm[:, 5], rec["flags"][sel], tm[:, 4] - tm[:, 3]):
            c = ctas.setdefault(int(k), [a, b, int(f), []])
            c[0], c[1] = min(c[0], a), max(c[1], b)
            c[3].append(int(st))
        durs = sorted(((v[1] - v[0]) / 1e3, k, v[2], max(v[3]) / 1e3, min(v[3]) / 1e3) for k, v in ctas.items())
        imb = np.array([max(v[3]) / max(1, min(v[3])) for v in ctas.values() if len(v[3]) > 1])
        if imb.size:  # slowest / fastest warp of a CTA in the states phase
            d["warp_imbalance"] = {"median": float(np.median(imb)), "p90": float(np.percentile(imb, 90)),
                                   "mean_busy_frac": float(np.mean([np.mean(v[3]) / max(v[3]) for v in ctas.values() if max(v[3]) > 0]))}
        d["ctas"] = len(ctas)
        d["cta_median_us"] = durs[len(durs) // 2][0]
        d["slowest"] = [{"us": u, "bx": k // 100000, "by": k % 100000, "fast": f & 1, "pin": (f >> 8) & 255,
                         "pfast": (f >> 16) & 255, "states_max_warp_us": smax, "states_min_warp_us": smin}
                        for u, k, f, smax, smin in durs[-6:]]
        d["start_offset_us"] = float((tm[:, 0].min() - t0) / 1e3)
        out["mode%d" % mode] = d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="paper")
    a = ap.parse_args()
    import torch
    from paper_2503_02412_b200 import se2map as S
    name = a.config
    c = CONFIGS[name]
    nx, ny, r, n_yaw = c["nx"], c["ny"], c["r"], c["n_yaw"]
    m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=c["robot"][0], robot_y=c["robot"][1])
    I, J = m.origin()
    m.update_elevation(world_heights(c["terrain"], I, J, nx, ny, r))
    m.assess_se2(0)
    m.synchronize()
    m.debug_phases(reset=True)
    if name != "stream":
        m.assess_se2(0)
        m.synchronize()
        print(json.dumps(summarize(m.debug_phases(), name + " FULL")))
        return
    path = robot_path(c["path_seed"], 60, r, *c["robot"])
    I0 = int(math.floor(path[:, 0].min() / r)) - nx // 2 - 2
    J0 = int(math.floor(path[:, 1].min() / r)) - ny // 2 - 2
    W = int(math.ceil((path[:, 0].max() - path[:, 0].min()) / r)) + nx + 6
    H = int(math.ceil((path[:, 1].max() - path[:, 1].min()) / r)) + ny + 6
    wh = torch.from_numpy(world_heights(c["terrain"], I0, J0, W, H, r)).cuda()
    for t in range(1, 40):
        m.step(*path[t], wh, I0, J0)
    m.synchronize()
    m.debug_phases(reset=True)
    for t in range(40, 41):
        m.step(*path[t], wh, I0, J0)
    m.synchronize()
    print(json.dumps(summarize(m.debug_phases(), "stream step")))


if __name__ == "__main__":
    main()
