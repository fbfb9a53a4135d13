"""GPU edge cases: empty inputs, degenerate footprints, many yaw bins, maximal clipping."""
import math

import numpy as np
import pytest

import oracle
from synth.terrain import CONFIGS, Hills, world_heights
from tests.gpu_common import make_map, oracle_params, run_config
from tests.parity import compare

pytestmark = pytest.mark.gpu


def test_empty_calls():
    """Zero-size rectangles, zero queries, zero points, a step without displacement: no work, no error."""
    import torch
    from paper_2503_02412_b200 import se2map as S
    m, h, g, orc, rep = run_config("tiny")
    m.update_elevation(np.zeros((0, 5), np.float32))
    q = m.query(np.zeros((0, 3)))
    assert len(q["risk"]) == 0
    pose = S.Pose.from_arrays(np.eye(3), np.zeros(3), np.eye(3), np.zeros(3), np.eye(3) * 1e-4,
                              np.zeros((3, 3)), np.zeros((3, 3)))
    cnt = m.integrate_scan(np.zeros((0, 3), np.float32), pose)
    assert list(cnt) == [0, 0, 0, 0, 0]
    x, y = CONFIGS["tiny"]["robot"]
    I_M, J_M = m.origin()
    world = torch.from_numpy(h).cuda()
    assert m.step(x, y, world, I_M, J_M) == (0, 0)
    m.assess_se2(1)                               # nothing dirty
    g2 = m.download()
    for f in g:
        assert np.array_equal(g[f], g2[f], equal_nan=True), f


@pytest.mark.parametrize("ex,ey", [(0.04, 0.04), (0.45, 0.04)])
def test_degenerate_stencils_are_unknown(ex, ey):
    """A footprint of fewer than 3 cells (|P| < 3, reading R8) or of one row of cells (collinear, R22)
    makes every state unknown: risk 1, trav 0, NaN angles — exactly as in the oracle."""
    nx, ny, r, n_yaw = 40, 36, 0.1, 8
    m = make_map(nx, ny, r, n_yaw, ex=ex, ey=ey)
    h = world_heights(Hills(seed=3), *m.origin(), nx, ny, r)
    m.update_elevation(h)
    m.assess_se2(0)
    g = m.download()
    orc = oracle.assess_all(oracle_params(nx, ny, r, n_yaw, ex, ey), h)
    rep = compare(g, orc)
    assert rep["ok"], rep
    assert rep["normal"] == 0 or (ex, ey) == (0.45, 0.04)  # a rotated line can cover 2-D cells at some angles


def test_many_yaw_bins():
    """360 bins (1-degree steps) on a small window: per-bin tables and pairing at scale."""
    cfg = dict(CONFIGS["paper"], nx=64, ny=56, n_yaw=360)
    m, h, g, orc, rep = run_config(cfg=cfg)
    print(rep)
    assert rep["ok"], rep


def test_window_of_one_row_and_column():
    """1 x n and n x 1 windows: every footprint is clipped to a line of cells — degenerate in the oracle
    (collinear, status 2) — and reported as unknown by the GPU (risk 1, trav 0, NaN angles; reading R22)."""
    for nx, ny in ((1, 40), (40, 1)):
        cfg = dict(CONFIGS["paper"], nx=nx, ny=ny, n_yaw=4)
        m, h, g, orc, rep = run_config(cfg=cfg)
        assert rep["ok"], rep
        assert rep["unknown"] + rep["ill"] == rep["n"] and rep["normal"] == 0
        assert np.all(np.isnan(g["pitch"])) and np.all(g["risk"] == 1) and np.all(g["trav"] == 0)


@pytest.mark.parametrize("robot", [(0.37, 0.61), (1.93, -0.44), (-3.05, 2.21)])
def test_vertical_edge_tiles_second_kernel(robot):
    """Tiles whose halo crosses only the window's left / right edge run in the column-major edge kernel
    on the edge stream (2 launches per assess when R_T <= 12): parity with the oracle on a tall window
    with unknown blobs next to both vertical edges (edge-kernel warps on the general path with holes
    inside the window, warps on the interior path, warps outside the window), traversable bits included,
    and INCREMENTAL after a sideways shift == FULL bit-exact."""
    nx, ny, r, n_yaw = 72, 200, 0.1, 16
    terrain = Hills(seed=17)
    m = make_map(nx, ny, r, n_yaw, robot=robot)
    I_M, J_M = m.origin()
    h = world_heights(terrain, I_M, J_M, nx, ny, r)
    rng = np.random.default_rng(11)
    known = np.ones((ny, nx), np.uint8)
    for _ in range(12):
        j = int(rng.integers(0, ny - 3))
        i = int(rng.choice([rng.integers(0, 6), rng.integers(nx - 6, nx - 1)]))
        known[j:j + 3, i:i + 2] = 0
    m.update_elevation(h, known)
    n0 = m.launch_count()
    m.assess_se2(0)
    assert m.launch_count() - n0 == 2                       # main kernel + edge kernel
    rep = compare(m.download(), oracle.assess_all(oracle_params(nx, ny, r, n_yaw), h, known))
    assert rep["ok"], rep
    # a sideways shift moves the window edges across tile columns; INCREMENTAL must equal FULL
    full = make_map(nx, ny, r, n_yaw, robot=robot)
    full.update_elevation(h, known)
    full.assess_se2(0)
    x, y = robot[0] + 0.57, robot[1]
    for mm in (m, full):
        di, dj = mm.shift_window(x, y)
    I_M, J_M = m.origin()
    h2 = world_heights(terrain, I_M, J_M, nx, ny, r)
    m.update_elevation(np.ascontiguousarray(h2[:, nx - di:]), i0=nx - di)
    full.update_elevation(h2, np.pad(known[:, di:], ((0, 0), (0, di)), constant_values=1))
    m.assess_se2(1)
    full.assess_se2(0)
    a, b = m.download(), full.download()
    for f in a:
        assert np.array_equal(a[f], b[f], equal_nan=True), f
