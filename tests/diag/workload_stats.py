#!/usr/bin/env python
"""Realised distributions of the synthetic workloads ("report the realised distributions per
config: trav fraction; early-return causes (kappa / pitch / roll); C12 and near-threshold counts"), from the
FP64 oracle (test infrastructure: this script lives under tests/).  CPU only.

    python tests/diag/workload_stats.py [--samples 200000] [--out profiles/workload_stats.json]

tiny / paper / the stream's first window: every state; high-res and large: a uniform random sample of states
(seeded).  Per config: states, |P_k| (gathered cells) mean / min, unknown (|P| < 3), ill-conditioned (oracle
degenerate, relative eigen-gap < 1e-3, or an angle > 1.3 rad: reading R12, excluded from parity), early
returns by cause (kappa > kappa_max; attitude: |pitch| > phi_x_max and / or |roll| > phi_y_max), near-threshold
states (within 1e-5 of a threshold), traversable fraction, risk quantiles of the traversable states.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth.terrain import CONFIGS, DEFAULT_RISK, world_heights  # noqa: E402
from tests.parity import classify  # noqa: E402


def stats(name, res, kappa_max, phi_x, phi_y):
    unknown, ill, near, normal = classify(res, kappa_max, phi_x, phi_y)
    st = res["status"]
    ok = st == 0
    with np.errstate(invalid="ignore"):
        early_k = ok & (res["early"] == 1)
        early_a = ok & (res["early"] == 2)
        px = ok & (np.abs(res["pitch"]) > phi_x)
        ry = ok & (np.abs(res["roll"]) > phi_y)
    trav = res["trav"] == 1
    n = int(res.size)
    risk_t = res["risk"][trav]
    out = {
        "config": name, "states": n,
        "cells_per_footprint_mean": float(res["n_points"][ok].mean()) if ok.any() else 0.0,
        "cells_per_footprint_min": int(res["n_points"].min()),
        "unknown": int(unknown.sum()), "ill_conditioned": int(ill.sum()), "near_threshold": int(near.sum()),
        "early_kappa": int(early_k.sum()), "early_attitude": int(early_a.sum()),
        "attitude_pitch_over": int((early_a & px).sum()), "attitude_roll_over": int((early_a & ry).sum()),
        "attitude_both_over": int((early_a & px & ry).sum()),
        "traversable_fraction": float(trav.mean()),
        "non_traversable_fraction": float(1.0 - trav.mean()),
        "risk_traversable_p10_p50_p90": [float(np.percentile(risk_t, q)) for q in (10, 50, 90)] if risk_t.size else [],
    }
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=200_000)
    ap.add_argument("--out")
    a = ap.parse_args()
    km, pxm, pym = DEFAULT_RISK["kappa_max"], DEFAULT_RISK["phi_x_max"], DEFAULT_RISK["phi_y_max"]
    rows = []
    for name in ("tiny", "paper", "stream", "highres", "large"):
        c = CONFIGS[name]
        nx, ny, r, n_yaw = c["nx"], c["ny"], c["r"], c["n_yaw"]
        I_M, J_M = oracle.window_origin(*c["robot"], r, nx, ny)
        h = world_heights(c["terrain"], I_M, J_M, nx, ny, r)
        prm = oracle.Params(nx=nx, ny=ny, resolution=r, n_yaw=n_yaw, ex=c["ex"], ey=c["ey"], **DEFAULT_RISK)
        t0 = time.time()
        if nx * ny * n_yaw <= 400_000:
            res = oracle.assess_all(prm, h).ravel()
            how = "every state"
        else:
            rng = np.random.default_rng(7)
            ijk = np.stack([rng.integers(0, nx, a.samples), rng.integers(0, ny, a.samples),
                            rng.integers(0, n_yaw, a.samples)], axis=1)
            res = oracle.assess_states(prm, h, ijk)
            how = "%d uniform random states (seed 7)" % a.samples
        s = stats(name, res, km, pxm, pym)
        s["sample"] = how
        s["oracle_s"] = round(time.time() - t0, 2)
        rows.append(s)
        print(json.dumps(s), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"note": __doc__.strip().splitlines()[0], "configs": rows}, f, indent=1)
            f.write("\n")


if __name__ == "__main__":
    main()
