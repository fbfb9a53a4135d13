"""Diagnostics: GPU-vs-oracle errors on a scan-built map (front-end + Alg. 1), binned by gap and |P|."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle
from oracle.frontend import FrontendParams, Pose, integrate_scan
from synth.lidar import scan
from synth.terrain import Hills
from tests.gpu_common import make_map, oracle_params
from tests.parity import classify
from paper_2503_02412_b200 import se2map as S

terrain = Hills(seed=21)
nx, ny, r, n_yaw = 100, 100, 0.1, 36
path = [(0.37, 0.61, 0.3), (0.81, 0.44, 0.1), (1.56, 0.9, 0.6), (1.57, 0.91, 0.6)]
m = make_map(nx, ny, r, n_yaw, robot=path[0][:2])
w = oracle.Window(nx, ny, r, *path[0][:2])
for f, (x, y, yaw) in enumerate(path):
    m.shift_window(x, y); w.shift(x, y)
    fr = scan(terrain, x, y, yaw, seed=100 + f, n_az=600)
    if f == 0: pass
    m.integrate_scan(fr.points_s, S.Pose.from_arrays(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S, fr.Sigma_R, fr.Sigma_B))
    integrate_scan(w, fr.points_s, Pose(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S, fr.Sigma_R, fr.Sigma_B), FrontendParams())
m.assess_se2(0)
g = m.download()
o = oracle.assess_all(oracle_params(nx, ny, r, n_yaw), w.heights, w.known)
unknown, ill, near, normal = classify(o)
err = np.maximum(np.abs(g["pitch"] - o["pitch"]), np.abs(g["roll"] - o["roll"]))
err = np.where(normal | near, err, 0)
print("known frac", w.known.mean())
for lo, hi in ((1e-3, 3e-3), (3e-3, 1e-2), (1e-2, 3e-2), (3e-2, 1e-1), (1e-1, 1)):
    sel = (normal | near) & (o["gap"] >= lo) & (o["gap"] < hi)
    if sel.any():
        print(f"gap [{lo},{hi}): n={sel.sum()} max={err[sel].max():.2e} p99.9={np.percentile(err[sel], 99.9):.2e} n>1e-5={(err[sel]>1e-5).sum()} n>1e-4={(err[sel]>1e-4).sum()}")
for lo, hi in ((3, 10), (10, 30), (30, 80), (80, 200)):
    sel = (normal | near) & (o["n_points"] >= lo) & (o["n_points"] < hi)
    if sel.any():
        print(f"N [{lo},{hi}): n={sel.sum()} max={err[sel].max():.2e} n>1e-4={(err[sel]>1e-4).sum()}")
idx = np.argsort(err.ravel())[::-1][:6]
for f in idx:
    k, j, i = np.unravel_index(f, err.shape)
    s = o[k, j, i]
    print(f"k={k} j={j} i={i} err={err[k,j,i]:.2e} N={s['n_points']} gap={s['gap']:.2e} lam={s['lam']} pitch={s['pitch']:.3f}")
dz = np.where(normal | near, np.abs(g["z"] - o["z"]), 0)
print("z errors: max", dz.max(), "n>1e-4", (dz > 1e-4).sum(), "n>5e-5", (dz > 5e-5).sum())
for f in np.argsort(dz.ravel())[::-1][:6]:
    k, j, i = np.unravel_index(f, dz.shape)
    s = o[k, j, i]
    print(f"k={k} j={j} i={i} dz={dz[k,j,i]:.2e} dang={err[k,j,i]:.2e} N={s['n_points']} gap={s['gap']:.2e} "
          f"pitch={s['pitch']:.3f} roll={s['roll']:.3f} lam={s['lam']}")
