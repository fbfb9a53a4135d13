#!/usr/bin/env python
"""Stream-step breakdown (H1 + H2 + H9): host wall time per C-ABI call and device time of the INCREMENTAL
assess, on bench.py's stream configuration (diagnostics)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import exposed_strips  # noqa: E402
from synth.terrain import CONFIGS, robot_path, world_heights  # noqa: E402
from paper_2503_02412_b200 import se2map as S  # noqa: E402

cfg = CONFIGS["stream"]
nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
stream = torch.cuda.Stream()
m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=cfg["robot"][0], robot_y=cfg["robot"][1],
             cuda_stream=stream.cuda_stream)
path = robot_path(cfg["path_seed"], 300, r, *cfg["robot"])
xs, ys = path[:, 0], path[:, 1]
I0 = int(math.floor(xs.min() / r)) - nx // 2 - 2
J0 = int(math.floor(ys.min() / r)) - ny // 2 - 2
Wd = int(math.ceil((xs.max() - xs.min()) / r)) + nx + 6
Hd = int(math.ceil((ys.max() - ys.min()) / r)) + ny + 6
wh = torch.from_numpy(world_heights(cfg["terrain"], I0, J0, Wd, Hd, r)).cuda()
with torch.cuda.stream(stream):
    I_M, J_M = m.origin()
    m.update_elevation(wh[J_M - J0:J_M - J0 + ny, I_M - I0:I_M - I0 + nx])
    m.assess_se2(0)
    stream.synchronize()
    t_shift, t_upd, t_ass, dev = [], [], [], []
    for t in range(1, len(path)):
        a = time.perf_counter()
        di, dj = m.shift_window(*path[t])
        b = time.perf_counter()
        I_M, J_M = m.origin()
        for (i0, j0, w, hh) in exposed_strips(di, dj, nx, ny):
            m.update_elevation(wh[J_M - J0 + j0:J_M - J0 + j0 + hh, I_M - I0 + i0:I_M - I0 + i0 + w], i0=i0, j0=j0)
        c = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m.assess_se2(1)
        e1.record(stream)
        d = time.perf_counter()
        stream.synchronize()
        if t > 20:
            t_shift.append(b - a); t_upd.append(c - b); t_ass.append(d - c); dev.append(e0.elapsed_time(e1))
print({"host_us_shift": 1e6 * np.median(t_shift), "host_us_updates": 1e6 * np.median(t_upd),
       "host_us_assess_call": 1e6 * np.median(t_ass), "device_us_assess": 1e3 * np.median(dev)})
