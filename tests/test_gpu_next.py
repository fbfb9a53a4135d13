"""GPU parity for the §8(f) NEXT rows built so far: NEXT-2 (SDF of the Risk = 1 set) and NEXT-3 (the
planner's trilinear Risk / SDF query with gradients), against the FP64 oracles (oracle.sdf,
oracle.trilinear) on the oracle's own inputs.
"""
import math

import numpy as np
import pytest

import oracle
from oracle.trilinear import trilinear
from synth.terrain import CONFIGS, Plane, world_heights
from tests.gpu_common import make_map, oracle_params, run_config
from tests.parity import classify

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,r,d_max,density", [((3, 70, 90), 0.1, 2.0, 0.1), ((2, 41, 37), 0.05, 0.8, 0.03),
                                                  ((1, 130, 64), 0.1, 9.6, 0.002), ((2, 20, 25), 0.1, 0.55, 0.5),
                                                  # column-pass segments (128 rows) and row-pass spans with
                                                  # ragged tails, W from 6 to 96 cells
                                                  ((2, 100, 530), 0.1, 2.0, 0.02), ((1, 140, 300), 0.1, 7.0, 0.005),
                                                  # rows longer than one row-pass CTA (1024 columns), ragged
                                                  ((1, 40, 2100), 0.1, 2.0, 0.02), ((1, 24, 1300), 0.1, 9.6, 0.002)])
def test_sdf_from_mask_matches_oracle(shape, r, d_max, density):
    from paper_2503_02412_b200 import se2map as S
    rng = np.random.default_rng(int(d_max * 100))
    mask = (rng.random(shape) < density).astype(np.uint8)
    mask[0, 5:12, 8:30] = 1
    if shape[0] > 1:
        mask[1] = 0                                   # a layer without obstacles: +d_max everywhere
    g = S.sdf_from_mask(mask, r, d_max)
    o = oracle.sdf(mask, r, d_max)
    assert np.max(np.abs(g - o)) <= 1e-6 * max(1.0, d_max)
    assert np.all((g < 0) == (mask == 1))


def test_map_sdf_and_trilinear_risk():
    """Map mode: the SDF follows the map's traversable bits through the ring buffer (after shifts);
    trilinear Risk / SDF queries agree with the oracle wherever the two obstacle sets agree."""
    cfg = dict(CONFIGS["paper"])
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    m = make_map(nx, ny, r, n_yaw, robot=cfg["robot"])
    I_M, J_M = m.origin()
    m.update_elevation(world_heights(cfg["terrain"], I_M, J_M, nx, ny, r))
    m.assess_se2(0)
    di, dj = m.shift_window(cfg["robot"][0] + 1.33, cfg["robot"][1] - 0.71)    # exercise the ring seam
    I_M, J_M = m.origin()
    h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
    m.update_elevation(h)
    m.assess_se2(1)
    d_max = 1.5
    m.compute_sdf(d_max)
    g = m.download()
    gs = m.download_sdf()
    orc = oracle.assess_all(oracle_params(nx, ny, r, n_yaw), h)
    mask_o = (orc["trav"] == 0).astype(np.uint8)
    so = oracle.sdf(mask_o, r, d_max)
    # cells whose (2W+1)^2 neighbourhood has the same obstacle set on both sides must agree exactly
    W = int(math.ceil(d_max / r))
    diff = (mask_o != (g["trav"] == 0)).astype(np.int32)
    k_bad = np.zeros_like(diff, dtype=bool)
    for k in range(n_yaw):
        ys, xs = np.nonzero(diff[k])
        for y, x in zip(ys, xs):
            k_bad[k, max(0, y - W):y + W + 1, max(0, x - W):x + W + 1] = True
    ok = ~k_bad
    assert ok.mean() > 0.9
    assert np.max(np.abs(gs[ok] - so[ok])) <= 1e-6 * d_max
    # trilinear: queries whose 8 corners are all 'normal' (risk) / unaffected (sdf)
    unknown, ill, near, normal = classify(orc)
    rng = np.random.default_rng(5)
    nq = 4000
    q = np.stack([rng.uniform((I_M + 0.5) * r, (I_M + nx - 0.5) * r, nq), rng.uniform((J_M + 0.5) * r, (J_M + ny - 0.5) * r, nq),
                  rng.uniform(-math.pi, math.pi, nq)], axis=1)
    vo, go_, oko = trilinear(orc["risk"], I_M, J_M, r, q)
    vs_o, gs_o, _ = trilinear(so, I_M, J_M, r, q)
    vg, gg, st = m.query_trilinear(q, 0)
    vsg, gsg, st2 = m.query_trilinear(q, 1)
    dth = 2 * math.pi / n_yaw
    n_cmp = 0
    for t in range(nq):
        if not oko[t]:
            assert np.isnan(vg[t])
            continue
        fx, fy = q[t, 0] / r - 0.5 - I_M, q[t, 1] / r - 0.5 - J_M
        i0, j0 = int(math.floor(fx)), int(math.floor(fy))
        k0 = int(math.floor((q[t, 2] + math.pi) / dth)) % n_yaw
        ks, js, is_ = [k0, (k0 + 1) % n_yaw], [j0, j0 + 1], [i0, i0 + 1]
        corners = [(k, j, i) for k in ks for j in js for i in is_]
        if all(normal[c] for c in corners):
            cmax = max(abs(orc["risk"][c]) for c in corners)
            tol = 1e-3 * cmax + 1e-5
            assert abs(vg[t] - vo[t]) <= tol, (t, vg[t], vo[t])
            assert np.all(np.abs(gg[t] - go_[t]) <= 8 * tol / np.array([r, r, dth]))
            n_cmp += 1
        if all(ok[c] for c in corners):
            assert abs(vsg[t] - vs_o[t]) <= 1e-5
            assert np.all(np.abs(gsg[t] - gs_o[t]) <= 1e-4 / np.array([r, r, dth]))
    # the asynchronous form with pinned host buffers (read / written in place by the kernel) and with device
    # buffers returns exactly the synchronous values
    import torch
    for field, (v_ref, g_ref) in ((0, (vg, gg)), (1, (vsg, gsg))):
        for dev in ("cpu", "cuda"):
            xt = torch.from_numpy(q.copy())
            xt = xt.pin_memory() if dev == "cpu" else xt.cuda()
            out = torch.full((4, nq), 7.0, dtype=torch.float32)
            out = out.pin_memory() if dev == "cpu" else out.cuda()
            m.query_trilinear_async(xt, out, field)
            m.synchronize()
            o = out.cpu().numpy()
            assert np.array_equal(o[0], v_ref, equal_nan=True), (field, dev)
            assert np.array_equal(o[1:].T, g_ref, equal_nan=True), (field, dev)
    assert n_cmp > 0.8 * nq


def test_trilinear_plane_closed_form():
    """On an exact plane the risk depends on theta only (closed form, pin Q2): the GPU interpolant
    matches the oracle interpolant of the oracle's risk to float precision, gradient in x, y ~ 0."""
    r, nx, ny, n = 0.125, 48, 40, 24
    m = make_map(nx, ny, r, n, ex=0.75, ey=0.5)
    I_M, J_M = m.origin()
    h = world_heights(Plane(gx=0.25, gy=-0.125, h0=64.0), I_M, J_M, nx, ny, r)
    m.update_elevation(h)
    m.assess_se2()
    orc = oracle.assess_all(oracle_params(nx, ny, r, n, 0.75, 0.5), h)
    rng = np.random.default_rng(6)
    q = np.stack([rng.uniform((I_M + 8) * r, (I_M + nx - 8) * r, 500), rng.uniform((J_M + 8) * r, (J_M + ny - 8) * r, 500),
                  rng.uniform(-4, 4, 500)], axis=1)
    vo, go_, oko = trilinear(orc["risk"], I_M, J_M, r, q)
    vg, gg, st = m.query_trilinear(q, 0)
    assert oko.all() and st == 0
    assert np.max(np.abs(vg - vo)) < 2e-6
    assert np.max(np.abs(gg[:, :2])) < 1e-4 and np.max(np.abs(gg[:, 2] - go_[:, 2])) < 2e-5


def test_sdf_requires_assess_and_rejects_bad_args():
    from paper_2503_02412_b200 import se2map as S
    m = make_map(20, 20, 0.1, 8)
    with pytest.raises(S.Se2mError) as e:
        m.compute_sdf(1.0)
    assert e.value.status == S.SE2M_ERR_STATE
    m.update_elevation(np.zeros((20, 20), np.float32))
    m.assess_se2()
    with pytest.raises(S.Se2mError):
        m.query_trilinear(np.zeros((1, 3)), 1)             # no SDF yet
    with pytest.raises(S.Se2mError) as e:
        m.compute_sdf(100.0)                               # 1000 cells > 96
    assert e.value.status == S.SE2M_ERR_UNSUPPORTED
    m.compute_sdf(0.5)
    s = m.download_sdf()
    assert np.all(s == np.float32(0.5))                    # flat: no obstacle anywhere
