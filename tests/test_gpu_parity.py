"""GPU parity: the CUDA path (through the C ABI) against the FP64 oracle, element by element.

Tolerances are the north_star's (tests/parity.py).  Run with -m gpu on a B200.
"""
import math

import numpy as np
import pytest

import oracle
from synth.terrain import CONFIGS, Hills, Plane, PlaneSine, world_heights
from tests.gpu_common import make_map, oracle_params, run_config
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _show(name, rep):
    print(name, {k: rep[k] for k in sorted(rep)})


@pytest.mark.parametrize("n_yaw", [9, 1, 72])
def test_parity_paper_window_yaw_counts(n_yaw):
    """Interior tiles (arrowhead solve) with odd n_yaw (no theta / theta + pi pairing), a single bin, and 5-degree
    bins, on the paper-like window."""
    m, h, gpu, orc, rep = run_config(cfg=dict(CONFIGS["paper"], n_yaw=n_yaw))
    _show("paper n_yaw=%d" % n_yaw, rep)
    assert rep["ok"], rep


@pytest.mark.parametrize("name", ["tiny", "tiny_small_fp", "paper"])
def test_parity_configs(name):
    m, h, gpu, orc, rep = run_config(name)
    _show(name, rep)
    assert rep["ok"], rep
    assert rep["normal"] > 0.5 * rep["n"] or name.startswith("tiny")


def test_parity_unknown_cells_and_holes():
    cfg = dict(CONFIGS["paper"])
    rng = np.random.default_rng(3)
    known = (rng.random((cfg["ny"], cfg["nx"])) > 0.1).astype(np.uint8)
    known[40:60, 10:30] = 0                                 # a big hole
    m, h, gpu, orc, rep = run_config(cfg=cfg, known=known)
    _show("holes", rep)
    assert rep["ok"], rep


@pytest.mark.parametrize("nx,ny,n_yaw,r,ex,ey", [
    (37, 23, 5, 0.1, 0.8, 0.5),       # odd n_yaw (no theta/theta+pi pairing), ragged tiles
    (50, 70, 1, 0.1, 0.45, 0.3),      # one yaw bin
    (64, 48, 12, 0.05, 0.8, 0.5),     # R = 16, window smaller than some halos
    (96, 40, 8, 0.1, 1.1, 0.35),      # R = 11 -> R_T = 12, nx % 32 == 0
    (9, 7, 4, 0.1, 0.3, 0.2),         # window smaller than a tile
])
def test_parity_shapes(nx, ny, n_yaw, r, ex, ey):
    cfg = dict(nx=nx, ny=ny, r=r, n_yaw=n_yaw, ex=ex, ey=ey, robot=(-1.37, 2.21), terrain=Hills(seed=7))
    m, h, gpu, orc, rep = run_config(cfg=cfg)
    _show("shape", rep)
    assert rep["ok"], rep


@pytest.mark.parametrize("c", [0.0, 2.5, 100.0])
def test_flat_plane_exact(c):
    """Pin Q1 on the GPU: a flat plane gives exactly zero pitch/roll/risk, z = c."""
    m = make_map(40, 36, 0.1, 8)
    h = np.full((36, 40), c, np.float32)
    m.update_elevation(h)
    m.assess_se2()
    g = m.download()
    orc = oracle.assess_all(oracle_params(40, 36, 0.1, 8), h)
    ok = orc["status"] == 0
    assert np.all(g["pitch"][ok] == 0) and np.all(g["roll"][ok] == 0) and np.all(g["risk"][ok] == 0)
    assert np.all(g["z"][ok] == c) and np.all(g["trav"][ok] == 1)


@pytest.mark.parametrize("gx,gy", [(0.375, -0.25), (0.75, 0.0), (-0.125, 0.5)])
def test_inclined_plane_closed_form(gx, gy):
    """Pin Q2 on the GPU: pitch/roll of an exact plane as a closed-form function of yaw."""
    r, nx, ny, n = 0.125, 48, 40, 12
    m = make_map(nx, ny, r, n, ex=0.75, ey=0.5)
    I_M, J_M = m.origin()
    h = world_heights(Plane(gx=gx, gy=gy, h0=64.0), I_M, J_M, nx, ny, r)
    m.update_elevation(h)
    m.assess_se2()
    g = m.download()
    alpha, beta = math.atan(math.hypot(gx, gy)), math.atan2(gy, gx)
    sa, ca = math.sin(alpha), math.cos(alpha)
    orc = oracle.assess_all(oracle_params(nx, ny, r, n, 0.75, 0.5), h)
    for k in range(n):
        th = -math.pi + 2 * math.pi * k / n
        den = math.sqrt(1 - sa * sa * math.cos(th - beta) ** 2)
        pitch = math.asin(ca * sa * math.cos(th - beta) / den)
        roll = math.asin(-sa * math.sin(th - beta) / den)
        ok = orc["status"][k] == 0
        assert np.max(np.abs(g["pitch"][k][ok] - pitch)) < 1e-5
        assert np.max(np.abs(g["roll"][k][ok] - roll)) < 1e-5


def test_theta_plus_pi_exact():
    """Pin Q3 on the GPU: bins k and k + n/2 differ only by the sign of pitch and roll (bit-exact)."""
    m, h, g, orc, rep = run_config("paper")
    H = 18
    a, b = slice(0, H), slice(H, 2 * H)
    for f in ("risk", "z", "trav"):
        assert np.array_equal(g[f][a], g[f][b], equal_nan=(f != "trav")), f
    assert np.array_equal(g["pitch"][a], -g["pitch"][b], equal_nan=True)
    assert np.array_equal(g["roll"][a], -g["roll"][b], equal_nan=True)


def test_device_pointer_update_matches_host():
    torch = pytest.importorskip("torch")
    cfg = CONFIGS["paper"]
    m1, h, g1, orc, rep = run_config("paper")
    m2 = make_map(cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"], robot=cfg["robot"])
    m2.update_elevation(torch.from_numpy(h).cuda())
    m2.assess_se2()
    g2 = m2.download()
    for f in g1:
        assert np.array_equal(g1[f], g2[f], equal_nan=True), f


def test_query_matches_download_and_oracle_index():
    m, h, g, orc, rep = run_config("paper")
    I_M, J_M = m.origin()
    rng = np.random.default_rng(9)
    n = 2000
    r, nx, ny, ny_aw = 0.1, 100, 100, 36
    xyt = np.stack([rng.uniform((I_M - 5) * r, (I_M + nx + 5) * r, n), rng.uniform((J_M - 5) * r, (J_M + ny + 5) * r, n),
                    rng.uniform(-4, 4, n)], axis=1)
    q = m.query(xyt)
    for t in range(n):
        idx = oracle.query_index(*xyt[t], I_M, J_M, nx, ny, r, ny_aw)
        if idx is None:
            assert np.isnan(q["risk"][t]) and q["trav"][t] == 0
            continue
        i, j, k = idx
        assert q["risk"][t] == g["risk"][k, j, i]
        assert q["trav"][t] == g["trav"][k, j, i]
        assert (q["pitch"][t] == g["pitch"][k, j, i]) or (np.isnan(q["pitch"][t]) and np.isnan(g["pitch"][k, j, i]))
    assert q["status"] != 0  # some queries were outside
    # the asynchronous form (pinned host buffers: read / written in place by the kernel; pageable NumPy buffers:
    # staged through device memory; device buffers) returns the same values
    import torch
    for dev in ("cpu", "numpy", "cuda"):
        if dev == "numpy":
            xt, out = xyt.copy(), np.full((5, n), 7.0, np.float32)
        else:
            xt = torch.from_numpy(xyt.copy())
            xt = xt.pin_memory() if dev == "cpu" else xt.cuda()
            out = torch.full((5, n), 7.0, dtype=torch.float32)
            out = out.pin_memory() if dev == "cpu" else out.cuda()
        m.query_async(xt, out)
        m.synchronize()
        o = out if dev == "numpy" else out.cpu().numpy()
        for row, f in enumerate(("risk", "pitch", "roll", "z")):
            assert np.array_equal(o[row], q[f], equal_nan=True), (dev, f)
        assert np.array_equal(o[4] > 0.5, q["trav"] == 1), dev


def test_errors():
    from paper_2503_02412_b200 import se2map as S
    with pytest.raises(S.Se2mError) as e:
        make_map(0, 10, 0.1, 8)
    assert e.value.status == S.SE2M_ERR_INVALID_ARG
    with pytest.raises(S.Se2mError) as e:
        make_map(10, 10, -0.1, 8)
    assert e.value.status == S.SE2M_ERR_INVALID_ARG
    m = make_map(20, 20, 0.1, 8)
    with pytest.raises(S.Se2mError) as e:
        m.assess_se2()                                     # before any elevation
    assert e.value.status == S.SE2M_ERR_STATE
    with pytest.raises(S.Se2mError) as e:
        m.update_elevation(np.zeros((5, 5), np.float32), i0=18, j0=0)
    assert e.value.status == S.SE2M_ERR_OUT_OF_RANGE


def test_all_unknown_after_big_shift():
    m, h, g, orc, rep = run_config("tiny")
    m.shift_window(1000.0, 1000.0)
    m.assess_se2(1)
    g2 = m.download()
    assert np.all(np.isnan(g2["pitch"])) and np.all(g2["risk"] == 1) and np.all(g2["trav"] == 0)


@pytest.mark.parametrize("nx,ny,robot", [(100, 100, (0.37, 0.61)), (37, 23, (-1.37, 2.21)), (64, 40, (5.55, -3.21))])
def test_download_compact_matches_download(nx, ny, robot):
    cfg = dict(CONFIGS["paper"], nx=nx, ny=ny, robot=robot)
    m, h, g, orc, rep = run_config(cfg=cfg)
    c = m.download_compact()
    assert c["risk_h"].dtype == np.float16
    assert np.array_equal(c["risk_h"], g["risk"].astype(np.float16))          # IEEE binary16, round to nearest
    # the planner's copy itself meets the north_star risk tolerance against the FP64 oracle
    rep_h = compare(dict(g, risk=c["risk_h"].astype(np.float32)), orc)
    assert rep_h["ok"], rep_h
    wpr = (nx + 31) // 32
    t = np.zeros((g["trav"].shape[0], ny, wpr * 32), np.uint64)
    t[:, :, :nx] = g["trav"]
    exp_bits = (t.reshape(-1, ny, wpr, 32) << np.arange(32, dtype=np.uint64)).sum(-1).astype(np.uint32)
    assert np.array_equal(c["trav_bits"], exp_bits)


@pytest.mark.parametrize("n_yaw", [36, 9])
def test_download_compact_rep_is_the_pi_periodic_half(n_yaw):
    """Representative planes (R13 / R23): risk and traversability of bins k and k + n/2 are identical, so
    the rep download equals the first n/2 planes of the full compact download AND its second half;
    asynchronous host copies into two buffers in flight, read after synchronize(); device destinations."""
    import torch
    cfg = dict(CONFIGS["paper"], n_yaw=n_yaw)
    m, h, g, orc, rep = run_config(cfg=cfg)
    full = m.download_compact()
    n_rep = n_yaw // 2 if n_yaw % 2 == 0 else n_yaw
    outs = []
    for _ in range(2):
        outs.append({"risk_h": torch.empty((n_rep, 100, 100), dtype=torch.float16).pin_memory(),
                     "trav_bits": torch.empty((n_rep, 100, 4), dtype=torch.int32).pin_memory()})
        m.download_compact_rep(out=outs[-1])
    m.synchronize()
    for o in outs:
        rq = o["risk_h"].numpy()
        tb = o["trav_bits"].numpy().view(np.uint32)
        assert np.array_equal(rq, full["risk_h"][:n_rep]) and np.array_equal(tb, full["trav_bits"][:n_rep])
        if n_yaw % 2 == 0:
            assert np.array_equal(rq, full["risk_h"][n_rep:]) and np.array_equal(tb, full["trav_bits"][n_rep:])
    dev = {"risk_h": torch.empty((n_rep, 100, 100), dtype=torch.float16, device="cuda"),
           "trav_bits": torch.empty((n_rep, 100, 4), dtype=torch.int32, device="cuda")}
    m.download_compact_rep(out=dev)
    m.synchronize()
    assert np.array_equal(dev["risk_h"].cpu().numpy(), full["risk_h"][:n_rep])
