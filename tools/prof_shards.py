#!/usr/bin/env python
"""Per-rank device time of the north_star's multi-GPU splits, ranks emulated one after another on ONE GPU.

    python tools/prof_shards.py [--reps 10]

large (2000 x 2000 x 72) in row bands (own rows + halo by device copies) and high-res (800 x 800 x 72) in yaw
slices (whole window; a slice starting inside a chain period replays the chain from its restart), G = 1, 2,
4, 8: the median CUDA-event time of each rank's FULL assess, run alone on the device.  max over ranks / the
G = 1 time is the work-balance bound of the strong-scaling efficiency (no NCCL time included).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from synth.terrain import CONFIGS, world_heights  # noqa: E402


def time_assess(m, stream, reps):
    with torch.cuda.stream(stream):
        for _ in range(2):
            m.assess_se2(0)
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m.assess_se2(0)
            b.record(stream)
            ts.append((a, b))
        stream.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ts]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--configs", default="large,highres")
    ap.add_argument("--segments", type=int, default=0, help="params.chain_segments (0 = auto)")
    a = ap.parse_args()
    from paper_2503_02412_b200 import se2map as S
    stream = torch.cuda.Stream()
    res = {}
    for name in a.configs.split(","):
        c = CONFIGS[name]
        nx, ny, r, n_yaw = c["nx"], c["ny"], c["r"], c["n_yaw"]
        mode = S.SE2M_SHARD_ROWS if name == "large" else S.SE2M_SHARD_YAW
        I_M = J_M = None
        h = None
        out = {}
        for G in (1, 2, 4, 8):
            kw = dict(shard_mode=mode, rank=0, world_size=G) if G > 1 else {}
            maps = []
            for g in range(G):
                kw2 = dict(kw, rank=g) if G > 1 else {}
                maps.append(S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=c["robot"][0],
                                     robot_y=c["robot"][1], cuda_stream=stream.cuda_stream,
                                     chain_segments=a.segments, **kw2))
            if h is None:
                I_M, J_M = maps[0].origin()
                h = world_heights(c["terrain"], I_M, J_M, nx, ny, r)
            for m in maps:
                m.update_elevation(h)           # (timing only: every rank gets the whole window)
            ms = [time_assess(m, stream, a.reps) for m in maps]
            out[G] = {"rank_ms": ms, "max_ms": max(ms), "balance_eff": None, "segments": maps[0].chain_segments()}
            for m in maps:
                m.close()
            torch.cuda.empty_cache()
        t1 = out[1]["max_ms"]
        for G, v in out.items():
            v["balance_eff"] = t1 / (G * v["max_ms"])
        res[name] = out
    print(json.dumps(res))


if __name__ == "__main__":
    main()
