import sys, os, json, math
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from synth.terrain import CONFIGS, world_heights
from paper_2503_02412_b200 import se2map as S
import bench
cfg = CONFIGS["large"]; nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
stream = torch.cuda.Stream()
positions, margin = bench.robot_positions(cfg, 40)
m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=positions[0][0], robot_y=positions[0][1], cuda_stream=stream.cuda_stream)
I0, J0 = m.origin(); WX, WY = nx + 2 * margin, ny + 2 * margin; WI0, WJ0 = I0 - margin, J0 - margin
wd = torch.from_numpy(world_heights(cfg["terrain"], WI0, WJ0, WX, WY, r)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
nq = 4096
qi = torch.zeros((nq, 3), dtype=torch.float64).pin_memory(); qo = torch.empty((5, nq), dtype=torch.float32).pin_memory()
res = {k: [] for k in ("shift", "update", "assess", "query", "total")}
with torch.cuda.stream(stream):
    for t in range(1, 36):
        x, y = positions[t]
        I, J = m.origin()
        qi[:, 0] = torch.from_numpy(np.random.uniform((I + 5) * r, (I + nx - 5) * r, nq)); qi[:, 1] = torch.from_numpy(np.random.uniform((J + 5) * r, (J + ny - 5) * r, nq))
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(stream); m.shift_window(x, y); ev[1].record(stream)
        I, J = m.origin(); v = wd[J - WJ0:J - WJ0 + ny, I - WI0:I - WI0 + nx]
        m.update_elevation(v); ev[2].record(stream)
        m.assess_se2(0); ev[3].record(stream)
        m.query_async(qi, qo); ev[4].record(stream)
        stream.synchronize()
        if t > 5:
            for k, (a, b) in zip(("shift", "update", "assess", "query"), zip(ev[:-1], ev[1:])): res[k].append(a.elapsed_time(b) * 1e3)
            res["total"].append(ev[0].elapsed_time(ev[4]) * 1e3)
print(json.dumps({k: round(float(np.median(v)), 2) for k, v in res.items()}))
