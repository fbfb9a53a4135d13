"""GPU-vs-oracle comparison with the acceptance rules of DESIGN.md §parity (north_star tolerances).

Per state, using the ORACLE's values to classify (the reference decides the class):
  * unknown (oracle status 1, |P| < 3): the GPU must also report unknown (NaN pitch, risk 1,
    trav 0) — an integer decision, bit-exact;
  * excluded, ill-conditioned: oracle status 2 (degenerate), or relative eigen-gap < 1e-3, or
    max(|pitch|, |roll|) > 1.3 rad (reading R12) — counted, not compared;
  * near-threshold: |kappa - kappa_max|, ||pitch| - phi_x_max| or ||roll| - phi_y_max| < 1e-5 —
    pitch/roll/z still compared, risk/trav counted separately;
  * otherwise: |d pitch|, |d roll| <= 1e-4 rad, |d z| <= 1e-4 m, |d risk| <= 1e-3 |risk| + 1e-6,
    trav bit-exact.
"""
from __future__ import annotations

import numpy as np

TOL_ANGLE = 1e-4
TOL_Z = 1e-4
TOL_RISK_REL = 1e-3
TOL_RISK_ABS = 1e-6
BAND = 1e-5
GAP_MIN = 1e-3
ANGLE_MAX = 1.3


def classify(orc, kappa_max=0.1, phi_x_max=0.52, phi_y_max=0.52):
    st = orc["status"]
    unknown = st == 1
    with np.errstate(invalid="ignore"):
        ill = (st == 2) | ((st == 0) & ((orc["gap"] < GAP_MIN) |
                                         (np.maximum(np.abs(orc["pitch"]), np.abs(orc["roll"])) > ANGLE_MAX)))
        near = (st == 0) & ~ill & ((np.abs(orc["kappa"] - kappa_max) < BAND) |
                                   (np.abs(np.abs(orc["pitch"]) - phi_x_max) < BAND) |
                                   (np.abs(np.abs(orc["roll"]) - phi_y_max) < BAND))
    normal = (st == 0) & ~ill & ~near
    return unknown, ill, near, normal


def compare(gpu: dict, orc: np.ndarray, kappa_max=0.1, phi_x_max=0.52, phi_y_max=0.52) -> dict:
    """gpu: dict of arrays (risk, pitch, roll, z, trav) with the same shape as the oracle array."""
    unknown, ill, near, normal = classify(orc, kappa_max, phi_x_max, phi_y_max)
    g = {k: np.asarray(v) for k, v in gpu.items()}
    rep = dict(n=int(orc.size), unknown=int(unknown.sum()), ill=int(ill.sum()), near=int(near.sum()),
               normal=int(normal.sum()))
    # unknown states: bit-exact class
    bad_unknown = unknown & ~(np.isnan(g["pitch"]) & (g["risk"] == 1.0) & (g["trav"] == 0))
    rep["bad_unknown"] = int(bad_unknown.sum())
    # the GPU must not call a state unknown that the oracle assessed normally
    rep["bad_spurious_unknown"] = int((normal & np.isnan(g["pitch"])).sum())
    cmp = normal | near
    with np.errstate(invalid="ignore"):
        dp = np.abs(g["pitch"] - orc["pitch"])[cmp]
        dr = np.abs(g["roll"] - orc["roll"])[cmp]
        dz = np.abs(g["z"] - orc["z"])[cmp]
        rk = np.abs(g["risk"] - orc["risk"])[normal]
        rtol = (TOL_RISK_REL * np.abs(orc["risk"]) + TOL_RISK_ABS)[normal]
    rep["max_dpitch"] = float(np.nanmax(dp)) if dp.size else 0.0
    rep["max_droll"] = float(np.nanmax(dr)) if dr.size else 0.0
    rep["max_dz"] = float(np.nanmax(dz)) if dz.size else 0.0
    rep["max_drisk"] = float(np.nanmax(rk)) if rk.size else 0.0
    rep["bad_pitch"] = int((~(dp <= TOL_ANGLE)).sum())
    rep["bad_roll"] = int((~(dr <= TOL_ANGLE)).sum())
    rep["bad_z"] = int((~(dz <= TOL_Z)).sum())
    rep["bad_risk"] = int((~(rk <= rtol)).sum())
    rep["bad_trav"] = int((g["trav"][normal] != orc["trav"][normal]).sum())
    rep["near_trav_mismatch"] = int((g["trav"][near] != orc["trav"][near]).sum())
    rep["trav_fraction"] = float(orc["trav"].mean())
    rep["ok"] = all(rep[k] == 0 for k in ("bad_unknown", "bad_spurious_unknown", "bad_pitch", "bad_roll",
                                           "bad_z", "bad_risk", "bad_trav"))
    return rep
