"""Diagnostics: the worst GPU-vs-oracle states of a config (run on the GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from synth.terrain import CONFIGS
from tests.gpu_common import run_config
from tests.parity import classify

for name, known in (("paper", None), ("holes", "holes")):
    cfg = dict(CONFIGS["paper"])
    kn = None
    if known:
        rng = np.random.default_rng(3)
        kn = (rng.random((cfg["ny"], cfg["nx"])) > 0.1).astype(np.uint8)
        kn[40:60, 10:30] = 0
    m, h, g, o, rep = run_config(cfg=cfg, known=kn)
    unknown, ill, near, normal = classify(o)
    err = np.maximum(np.abs(g["pitch"] - o["pitch"]), np.abs(g["roll"] - o["roll"]))
    err = np.where(normal | near, err, 0)
    idx = np.argsort(err.ravel())[::-1][:8]
    print(name, rep["max_dpitch"], rep["max_droll"])
    for f in idx:
        k, j, i = np.unravel_index(f, err.shape)
        s = o[k, j, i]
        print(f"  k={k} j={j} i={i} err={err[k,j,i]:.2e} np={s['n_points']} gap={s['gap']:.3e} kappa={s['kappa']:.4f} "
              f"pitch={s['pitch']:.4f} roll={s['roll']:.4f} lam={s['lam']} n={s['n']}")
    # error vs gap histogram
    for lo_, hi_ in ((1e-3, 1e-2), (1e-2, 1e-1), (1e-1, 1)):
        sel = (normal | near) & (o["gap"] >= lo_) & (o["gap"] < hi_)
        if sel.any():
            print(f"  gap in [{lo_},{hi_}): n={sel.sum()} max err={err[sel].max():.2e} p99={np.percentile(err[sel],99):.2e}")
