"""GPU parity of NEXT-4 nearest-neighbour inpainting (se2m_inpaint, reading R31) against oracle/inpaint.py
(bit-exact: the view is a copy of known heights chosen by an integer rule), and of the whole pipeline
(inpaint -> Algorithm 1) against the oracle's assessment of the oracle's inpainted map."""
import numpy as np
import pytest

import oracle
from oracle.inpaint import inpaint_nearest
from synth.terrain import Hills, world_heights
from tests.gpu_common import make_map, oracle_params
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _blobs(rng, ny, nx, frac, size=3):
    """known mask with unknown blobs of size x size covering about frac of the window."""
    k = np.ones((ny, nx), np.uint8)
    nb = int(frac * nx * ny / size ** 2)
    cj, ci = rng.integers(0, ny, nb), rng.integers(0, nx, nb)
    for dj in range(size):
        for di in range(size):
            k[np.clip(cj + dj, 0, ny - 1), np.clip(ci + di, 0, nx - 1)] = 0
    return k


@pytest.mark.parametrize("nx,ny,frac,seed", [(37, 29, 0.5, 0), (100, 100, 0.9, 1), (130, 70, 0.99, 2),
                                             (64, 96, 0.3, 3)])
def test_inpaint_bit_exact(nx, ny, frac, seed):
    rng = np.random.default_rng(seed)
    r = 0.1
    m = make_map(nx, ny, r, 8, robot=(1.234, -2.71))
    I_M, J_M = m.origin()
    h = world_heights(Hills(seed=seed), I_M, J_M, nx, ny, r)
    known = (rng.random((ny, nx)) > frac).astype(np.uint8) if frac > 0.9 else _blobs(rng, ny, nx, frac)
    known[rng.integers(ny), rng.integers(nx)] = 1
    m.update_elevation(h, known)
    m.inpaint()
    g = m.download_inpainted()
    o, _ = inpaint_nearest(h, known)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def test_inpaint_after_shifts_ring_seam():
    """The view is computed in logical window coordinates across the ring seam (after shifts)."""
    rng = np.random.default_rng(7)
    nx, ny, r = 90, 70, 0.1
    terrain = Hills(seed=9)
    m = make_map(nx, ny, r, 8, robot=(0.37, 0.61))
    w = oracle.Window(nx, ny, r, 0.37, 0.61)
    for step, (x, y) in enumerate([(0.37, 0.61), (1.93, 0.12), (3.01, 2.47), (2.2, 3.9)]):
        m.shift_window(x, y)
        w.shift(x, y)
        I_M, J_M = m.origin()
        assert (I_M, J_M) == (w.I_M, w.J_M)
        h = world_heights(terrain, I_M, J_M, nx, ny, r)
        known = (rng.random((ny, nx)) > 0.8).astype(np.uint8)
        m.update_elevation(h, known)
        w.heights[:] = h
        w.known[:] = known
        g = m.download_inpainted()
        o, _ = inpaint_nearest(w.heights, w.known)
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32)), step


def test_inpaint_single_cell_and_all_unknown():
    m = make_map(40, 30, 0.1, 8)
    h = np.full((30, 40), np.nan, np.float32)
    h[11, 27] = 12.5
    m.update_elevation(h)
    assert np.all(m.download_inpainted() == np.float32(12.5))
    m2 = make_map(40, 30, 0.1, 8)
    m2.update_elevation(np.full((30, 40), np.nan, np.float32))
    with pytest.raises(RuntimeError):
        m2.inpaint()
    assert np.all(np.isnan(m2.download_inpainted()))


def test_pipeline_inpaint_assess_parity_and_incremental():
    """params.inpaint = 1: assess reads the view; parity vs the oracle on the oracle's inpainted map;
    then new measurements (a known patch) -> INCREMENTAL equals FULL bit-exactly."""
    rng = np.random.default_rng(11)
    nx, ny, r, n_yaw = 100, 100, 0.1, 36
    m = make_map(nx, ny, r, n_yaw, inpaint=1)
    I_M, J_M = m.origin()
    h = world_heights(Hills(seed=13), I_M, J_M, nx, ny, r)
    known = _blobs(rng, ny, nx, 0.6, size=5)
    m.update_elevation(h, known)
    m.assess_se2(0)
    g = m.download()
    hi, _ = inpaint_nearest(h, known)
    orc = oracle.assess_all(oracle_params(nx, ny, r, n_yaw), hi)
    rep = compare(g, orc)
    print(rep)
    assert rep["ok"], rep
    # a 12 x 9 patch becomes known: the view changes around it; INCREMENTAL must equal FULL
    patch = np.ascontiguousarray(h[40:49, 50:62])
    m.update_elevation(patch, i0=50, j0=40)
    m.assess_se2(1)
    inc = m.download()
    m.assess_se2(0)
    full = m.download()
    for key in ("risk", "pitch", "roll", "z", "trav"):
        assert np.array_equal(np.asarray(inc[key]).view(np.uint8), np.asarray(full[key]).view(np.uint8)), key
