"""Pins for the FP64 oracle: what the paper and the mathematics fix (Q1-Q12).

Each test pins the oracle to something other than itself: a closed form, an invariant of
the mathematics, a hand-derived worked example (tests/golden/), a textbook routine, or an
independent brute force (tests/bruteforce.py).  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from synth.terrain import Hills, Plane, PlaneSine, world_heights
from tests import bruteforce

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _window(terrain, nx, ny, r, I_M=-7, J_M=3):
    return world_heights(terrain, I_M, J_M, nx, ny, r), I_M, J_M


# ---- Q1: flat plane -> exact zeros everywhere, clipped borders included ---------------
@pytest.mark.parametrize("c", [0.0, 2.5, 100.0])
def test_q1_flat_plane_exact(c):
    P = oracle.Params(nx=18, ny=14, resolution=0.1, n_yaw=8)
    h = np.full((P.ny, P.nx), c, dtype=np.float32)
    res = oracle.assess_all(P, h)
    ok = res["status"] == 0
    assert ok.sum() > 0.9 * ok.size
    for f in ("pitch", "roll", "kappa", "risk"):
        assert np.all(res[f][ok] == 0.0), f
    assert np.all(res["z"][ok] == c)
    assert np.all(res["trav"][ok] == 1)
    # the states that are not 'ok' must be genuinely degenerate (< 3 points or collinear)
    for k, j, i in zip(*np.nonzero(~ok)):
        assert res["n_points"][k, j, i] < 3 or res["status"][k, j, i] == 2


# ---- Q2: inclined plane, closed form as a function of yaw (clipped footprints too) -----
def _plane_closed_form(gx, gy, theta):
    alpha = math.atan(math.hypot(gx, gy))
    beta = math.atan2(gy, gx)
    sa, ca = math.sin(alpha), math.cos(alpha)
    den = math.sqrt(1.0 - sa * sa * math.cos(theta - beta) ** 2)
    pitch = math.asin(ca * sa * math.cos(theta - beta) / den)
    roll = math.asin(-sa * math.sin(theta - beta) / den)
    return pitch, roll


@pytest.mark.parametrize("gx,gy", [(0.375, -0.25), (0.75, 0.0), (-0.125, 0.5), (0.0, 0.0)])
def test_q2_inclined_plane_closed_form(gx, gy):
    r = 0.125                                   # dyadic resolution -> exact float32 heights
    P = oracle.Params(nx=16, ny=12, resolution=r, n_yaw=12, ex=0.75, ey=0.5)
    plane = Plane(gx=gx, gy=gy, h0=64.0)
    h, I_M, J_M = _window(plane, P.nx, P.ny, r)
    assert np.array_equal(h.astype(np.float64),
                          64.0 + gx * (np.arange(I_M, I_M + P.nx)[None, :] + 0.5) * r
                          + gy * (np.arange(J_M, J_M + P.ny)[:, None] + 0.5) * r)
    res = oracle.assess_all(P, h)
    for k in range(P.n_yaw):
        th = -math.pi + 2 * math.pi * k / P.n_yaw
        pitch, roll = _plane_closed_form(gx, gy, th)
        ok = res["status"][k] == 0
        assert ok.sum() > 0.8 * ok.size
        assert np.max(np.abs(res["pitch"][k][ok] - pitch)) < 1e-12
        assert np.max(np.abs(res["roll"][k][ok] - roll)) < 1e-12
        assert np.max(np.abs(res["kappa"][k][ok])) < 1e-12
        xc = (np.arange(I_M, I_M + P.nx)[None, :] + 0.5) * r
        yc = (np.arange(J_M, J_M + P.ny)[:, None] + 0.5) * r
        zc = np.broadcast_to(64.0 + gx * xc + gy * yc, (P.ny, P.nx))
        assert np.max(np.abs(res["z"][k][ok] - zc[ok])) < 1e-11
        over = abs(pitch) > 0.52 or abs(roll) > 0.52
        if over:
            assert np.all(res["risk"][k][ok] == 1.0) and np.all(res["trav"][k][ok] == 0)
        else:
            exp = 0.3 * abs(pitch) / 0.52 + 0.3 * abs(roll) / 0.52
            assert np.max(np.abs(res["risk"][k][ok] - exp)) < 1e-11
            assert np.all(res["trav"][k][ok] == 1)


@pytest.mark.parametrize("ex", GOLDEN["alg1_planes"])
def test_q2_worked_examples_golden(ex):
    """SPEC.md:236-238 hand-derived Alg. 1 values (tests/golden/worked_examples.json)."""
    r = 0.1
    P = oracle.Params(nx=24, ny=24, resolution=r, n_yaw=8, w=tuple(ex["w"]), kappa_max=ex["kappa_max"])
    a = ex["alpha"]
    h, _, _ = _window(Plane(gx=math.tan(a), gy=0.0, h0=10.0), P.nx, P.ny, r)
    k = 4                                         # theta_4 = -pi + pi = 0
    assert -math.pi + 2 * math.pi * k / P.n_yaw == ex["theta"]
    s = oracle.assess_state(P, h, 12, 12, k)
    assert s["status"] == 0
    # float32 heights: tolerance from rounding the plane to float32 (~1e-7 relative)
    assert abs(s["risk"] - ex["risk"]) < 2e-6
    assert np.max(np.abs(np.array(s["n"]) - ex["nb"])) < 2e-6
    assert s["trav"] == ex["trav"]


# ---- Q3: theta vs theta + pi -> pitch/roll negated exactly, the rest equal --------------
def test_q3_theta_plus_pi_exact():
    P = oracle.Params(nx=30, ny=26, resolution=0.1, n_yaw=8)
    h, _, _ = _window(Hills(seed=11), P.nx, P.ny, P.resolution)
    res = oracle.assess_all(P, h)
    half = P.n_yaw // 2
    for k in range(half):
        a, b = res[k], res[k + half]
        ok = a["status"] == 0
        assert np.array_equal(a["status"], b["status"])
        assert np.array_equal(a["pitch"][ok], -b["pitch"][ok])
        assert np.array_equal(a["roll"][ok], -b["roll"][ok])
        for f in ("z", "kappa", "risk", "trav", "n_points"):
            assert np.array_equal(a[f][ok], b[f][ok]), f


# ---- Q4: translation invariance of the window ---------------------------------------------
def test_q4_translation_invariance():
    P = oracle.Params(nx=40, ny=36, resolution=0.1, n_yaw=6)
    t = Hills(seed=12)
    hA, IA, JA = _window(t, P.nx, P.ny, P.resolution, I_M=-10, J_M=5)
    hB, IB, JB = _window(t, P.nx, P.ny, P.resolution, I_M=-3, J_M=1)
    rA, rB = oracle.assess_all(P, hA), oracle.assess_all(P, hB)
    R = 9
    n_cmp = 0
    for J in range(max(JA, JB) + R, min(JA, JB) + P.ny - R):
        for I in range(max(IA, IB) + R, min(IA, IB) + P.nx - R):
            a = rA[:, J - JA, I - IA]
            b = rB[:, J - JB, I - IB]
            assert a.tobytes() == b.tobytes()
            n_cmp += 1
    assert n_cmp > 10


# ---- Q5: independent brute force on tiny grids -----------------------------------------
@pytest.mark.parametrize("cfg", ["sine", "hills", "holes"])
def test_q5_bruteforce(cfg):
    r, nx, ny, n_yaw, ex, ey = 0.1, 20, 16, 8, 0.8, 0.5
    if cfg == "sine":
        h, _, _ = _window(PlaneSine(), nx, ny, r)
        known = None
    else:
        h, _, _ = _window(Hills(seed=13), nx, ny, r)
        known = None
        if cfg == "holes":
            rng = np.random.default_rng(5)
            known = (rng.random((ny, nx)) > 0.2).astype(np.uint8)
    P = oracle.Params(nx=nx, ny=ny, resolution=r, n_yaw=n_yaw, ex=ex, ey=ey)
    res = oracle.assess_all(P, h, known)
    n_cmp = 0
    for k in range(n_yaw):
        for j in range(ny):
            for i in range(nx):
                bf = bruteforce.assess_state(h, known, i, j, k, r, n_yaw, ex, ey)
                if bf["tie"]:
                    continue
                o = res[k, j, i]
                assert o["n_points"] == bf["n_points"]
                assert o["status"] == bf["status"]
                if bf["status"] != 0:
                    continue
                if bf["gap"] < 1e-6:          # eigenvector ill-posed; both sides valid
                    continue
                for f in ("pitch", "roll", "z", "kappa", "risk"):
                    assert abs(o[f] - bf[f]) < 1e-10 * max(1.0, abs(bf[f])), (f, k, j, i, o[f], bf[f])
                assert o["trav"] == bf["trav"]
                n_cmp += 1
    assert n_cmp > 0.85 * n_yaw * nx * ny


# ---- Q6: eigen-solver vs characteristic-polynomial roots -------------------------------
def test_q6_eigen_vs_charpoly():
    rng = np.random.default_rng(6)
    for _ in range(1000):
        X = rng.normal(size=(3, 3)) * rng.uniform(0.01, 10, size=3)
        A = X @ X.T
        lam, V = oracle.eig3(A)
        tr = np.trace(A)
        m2 = A[0, 0] * A[1, 1] - A[0, 1] ** 2 + A[0, 0] * A[2, 2] - A[0, 2] ** 2 + A[1, 1] * A[2, 2] - A[1, 2] ** 2
        roots = np.sort(np.real(np.roots([1.0, -tr, m2, -np.linalg.det(A)])))
        scale = np.abs(A).max()
        assert np.max(np.abs(lam - roots)) < 1e-9 * scale
        assert np.max(np.abs(A @ V - V * lam)) < 1e-12 * scale
        assert np.max(np.abs(V.T @ V - np.eye(3))) < 1e-13
        assert lam[0] <= lam[1] <= lam[2]


# ---- Q7: scale invariance (power-of-two scale -> bit-exact) --------------------------------
@pytest.mark.parametrize("c", [2.0, 0.5, 4.0])
def test_q7_scale_invariance(c):
    r, nx, ny = 0.1, 22, 18
    P1 = oracle.Params(nx=nx, ny=ny, resolution=r, n_yaw=8, ex=0.8, ey=0.5)
    Pc = oracle.Params(nx=nx, ny=ny, resolution=r * c, n_yaw=8, ex=0.8 * c, ey=0.5 * c)
    h, _, _ = _window(Hills(seed=14), nx, ny, r)
    hc = (h.astype(np.float64) * c).astype(np.float32)
    assert np.array_equal(hc.astype(np.float64), h.astype(np.float64) * c)
    a, b = oracle.assess_all(P1, h), oracle.assess_all(Pc, hc)
    ok = a["status"] == 0
    assert np.array_equal(a["status"], b["status"])
    for f in ("pitch", "roll", "kappa", "risk", "trav"):
        assert np.array_equal(a[f][ok], b[f][ok]), f
    assert np.array_equal(a["z"][ok] * c, b["z"][ok])


# ---- Q8: tap-order invariance ------------------------------------------------------------
def test_q8_tap_order_invariance():
    P = oracle.Params(nx=24, ny=24, resolution=0.1, n_yaw=8)
    h, _, _ = _window(Hills(seed=15), P.nx, P.ny, P.resolution)
    rng = np.random.default_rng(8)
    for _ in range(40):
        i, j, k = int(rng.integers(0, 24)), int(rng.integers(0, 24)), int(rng.integers(0, 8))
        a = oracle.assess_state(P, h, i, j, k)
        if a["status"] != 0 or a["gap"] < 1e-6:
            continue
        for seed in (1, 2, 3):
            b = oracle.assess_state(P, h, i, j, k, shuffle_seed=seed)
            for f in ("pitch", "roll", "z", "kappa", "risk"):
                assert abs(a[f] - b[f]) < 1e-13 * max(1.0, abs(a[f])), f
            assert a["trav"] == b["trav"]


# ---- Q9: Eq. 4 worked examples (recentre) and window shift semantics -------------------------
@pytest.mark.parametrize("ex", GOLDEN["eq4_recentre"])
def test_q9_eq4_examples(ex):
    I_M, J_M = oracle.window_origin(ex["x"], ex["y"], ex["r"], 10, 10)
    assert (I_M + 5, J_M + 5) == (ex["I"], ex["J"])


def test_q9_shift_semantics():
    w = oracle.Window(12, 10, 0.1, 0.55, 0.55)
    w.heights[:] = np.arange(120, dtype=np.float32).reshape(10, 12)
    w.known[:] = 1
    h0, k0 = w.heights.copy(), w.known.copy()
    assert w.shift(0.55, 0.55) == (0, 0)                       # zero displacement: unchanged
    assert np.array_equal(w.heights, h0) and np.array_equal(w.known, k0)
    assert w.shift(0.55, 0.55) == (0, 0)                       # idempotent
    di, dj = w.shift(0.75, 0.45)                               # +2 cells in x, -1 in y
    assert (di, dj) == (2, -1)
    assert np.array_equal(w.heights[1:, :-2], h0[:-1, 2:])     # retained cells bit-exact
    assert not w.known[0, :].any() and not w.known[:, -2:].any()
    w.shift(100.0, 100.0)                                      # displacement >= side: all unknown
    assert not w.known.any()


# ---- Q10: bounds ------------------------------------------------------------------------------
def test_q10_bounds():
    P = oracle.Params(nx=30, ny=30, resolution=0.1, n_yaw=8)
    for seed in (21, 22):
        h, _, _ = _window(Hills(seed=seed, slope_rms=0.6), P.nx, P.ny, P.resolution)
        res = oracle.assess_all(P, h)
        ok = res["status"] == 0
        assert np.all((res["risk"] >= 0) & (res["risk"] <= 1))
        assert np.all((res["kappa"][ok] >= 0) & (res["kappa"][ok] <= 1.0 / 3.0 + 1e-15))
        assert np.all(res["risk"][~ok] == 1.0) and np.all(res["trav"][~ok] == 0)
        assert np.all(res["risk"][res["trav"] == 0] == 1.0)


# ---- Q12: phi_x = alpha on planes at 0.05 m, ellipse 0.8 x 0.5 ---------------------
@pytest.mark.parametrize("alpha", [0.0, 0.1, 0.2, 0.3, 0.4, 0.5])
def test_q12_pitch_equals_slope(alpha):
    r = 0.05
    P = oracle.Params(nx=40, ny=40, resolution=r, n_yaw=8, ex=0.8, ey=0.5)
    beta = 0.0
    h, _, _ = _window(Plane(gx=math.tan(alpha), gy=0.0, h0=5.0), P.nx, P.ny, r)
    s = oracle.assess_state(P, h, 20, 20, 4)                   # theta_4 = 0 = beta
    assert abs(s["pitch"] - alpha) < 1e-6 and abs(s["roll"]) < 1e-6
    assert beta == 0.0


# ---- query index (reading R3 / R6) ---------------------------------------------------------------
def test_query_index():
    assert oracle.query_index(0.05, 0.05, 0.0, 0, 0, 10, 10, 0.1, 8) == (0, 0, 4)
    assert oracle.query_index(-0.01, 0.05, 0.0, 0, 0, 10, 10, 0.1, 8) is None
    # theta = pi wraps to bin 0 (theta_0 = -pi)
    assert oracle.query_index(0.05, 0.05, math.pi, 0, 0, 10, 10, 0.1, 8)[2] == 0
    # nearest bin: theta just below -pi + dtheta/2 -> bin 0, just above -> bin 1
    d = 2 * math.pi / 8
    assert oracle.query_index(0.05, 0.05, -math.pi + 0.49 * d, 0, 0, 10, 10, 0.1, 8)[2] == 0
    assert oracle.query_index(0.05, 0.05, -math.pi + 0.51 * d, 0, 0, 10, 10, 0.1, 8)[2] == 1
