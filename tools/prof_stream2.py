#!/usr/bin/env python
"""se2m_step device time per step (CUDA events on the map's stream), with and without the CUDA-graph step
(params.step_graph), over the bench's stream configuration: mean / p50 / p99 microseconds over N steps."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.terrain import CONFIGS, robot_path, world_heights  # noqa: E402
from paper_2503_02412_b200 import se2map as S  # noqa: E402


def run(step_graph, n_steps=1000, warm=20):
    cfg = CONFIGS["stream"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    stream = torch.cuda.Stream()
    m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=cfg["robot"][0], robot_y=cfg["robot"][1],
                 cuda_stream=stream.cuda_stream, step_graph=step_graph)
    path = robot_path(cfg["path_seed"], n_steps + warm + 1, r, *cfg["robot"])
    I0 = int(math.floor(path[:, 0].min() / r)) - nx // 2 - 2
    J0 = int(math.floor(path[:, 1].min() / r)) - ny // 2 - 2
    W = int(math.ceil((path[:, 0].max() - path[:, 0].min()) / r)) + nx + 6
    H = int(math.ceil((path[:, 1].max() - path[:, 1].min()) / r)) + ny + 6
    wh = torch.from_numpy(world_heights(cfg["terrain"], I0, J0, W, H, r)).cuda()
    I, J = m.origin()
    with torch.cuda.stream(stream):
        m.update_elevation(world_heights(cfg["terrain"], I, J, nx, ny, r))
        m.assess_se2(0)
        ev = []
        for t in range(1, len(path)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m.step(*path[t], wh, I0, J0)
            b.record(stream)
            if t > warm:
                ev.append((a, b))
        stream.synchronize()
    us = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    m.close()
    return {"step_graph": step_graph, "steps": len(us), "mean_us": float(us.mean()), "p50_us": float(np.median(us)),
            "p99_us": float(np.percentile(us, 99))}


if __name__ == "__main__":
    for g in (0, 1, 0, 1):
        print(json.dumps(run(g)))
