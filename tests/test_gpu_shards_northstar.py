"""The north_star's multi-GPU splits at their own sizes (BASELINE.json configs), G = 2, 4, 8 ranks emulated as
independent handles on one GPU (Q13: sharded == single, bit-exact):

* large map 2000 x 2000 x 72 @ 0.1 m in interleaved tile-row bands: every rank is fed ONLY its own rows, the
  halo slabs (se2m_halo_pack / _unpack — the buffers se2m_exchange_halo sends with NCCL) are handed over by
  device copies (no rank waits on another: safe on one device); FULL, then INCREMENTAL after window shifts;
* high-res 800 x 800 x 72 @ 0.05 m in yaw slices: every rank is fed the whole window and assesses its bins
  (a slice starting inside a yaw-chain period replays the chain from the restart); FULL and INCREMENTAL.

Every rank's owned states must equal the unsharded map's bit for bit (compared on the device, all planes).
"""
import numpy as np
import pytest
import torch

from synth.terrain import CONFIGS, world_heights
from tests.gpu_common import make_map
from tests.test_gpu_halo import _runs
from tests.test_gpu_stream import _exposed_strips

pytestmark = pytest.mark.gpu

PLANES = ("risk", "pitch", "roll", "z", "trav")


def _dev_planes(m, shape):
    out = {f: torch.empty(shape, dtype=torch.uint8 if f == "trav" else torch.float32, device="cuda") for f in PLANES}
    m.download(out=out)
    return out


def _same_bits(a, b):
    if a.dtype == torch.float32:
        return torch.equal(a.view(torch.int32), b.view(torch.int32))
    return torch.equal(a, b)


def _check_rows(maps, single, J_M, shape):
    ref = _dev_planes(single, shape)
    G = len(maps)
    for g, m in enumerate(maps):
        TY = m.tile_info()[1]
        own = torch.from_numpy((np.floor_divide(np.arange(J_M, J_M + shape[1]), TY) % G) == g).cuda()
        got = _dev_planes(m, shape)
        for f in PLANES:
            assert _same_bits(got[f][:, own, :], ref[f][:, own, :]), (G, g, f)
        del got
    return True


def _exchange(maps):
    G = len(maps)
    cap, rows = maps[0].halo_size()
    nx = maps[0].params.nx
    to_lo, to_hi = [], []
    for m in maps:
        a = torch.empty((cap, rows, nx), dtype=torch.float32, device="cuda")
        b = torch.empty_like(a)
        m.halo_pack(-1, a)
        m.halo_pack(+1, b)
        m.synchronize()
        to_lo.append(a)
        to_hi.append(b)
    for g, m in enumerate(maps):
        m.halo_unpack(to_lo[(g + 1) % G], +1)
        m.halo_unpack(to_hi[(g - 1) % G], -1)
        m.synchronize()


@pytest.fixture(scope="module")
def large_world():
    cfg = CONFIGS["large"]
    probe = make_map(cfg["nx"], cfg["ny"], cfg["r"], 8, robot=cfg["robot"])
    I_M, J_M = probe.origin()
    probe.close()
    margin = 40
    W0, J0 = I_M - margin, J_M - margin
    h = world_heights(cfg["terrain"], W0, J0, cfg["nx"] + 2 * margin, cfg["ny"] + 2 * margin, cfg["r"])
    return W0, J0, h


@pytest.mark.parametrize("G", [2, 4, 8])
def test_large_row_bands_equal_single(G, large_world):
    cfg = CONFIGS["large"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    W0, J0, world = large_world
    robot = cfg["robot"]
    single = make_map(nx, ny, r, n_yaw, robot=robot)
    maps = [make_map(nx, ny, r, n_yaw, robot=robot, shard_mode=2, rank=g, world_size=G) for g in range(G)]
    try:
        I_M, J_M = single.origin()

        def win(I, J):
            return world[J - J0:J - J0 + ny, I - W0:I - W0 + nx]

        h = np.ascontiguousarray(win(I_M, J_M))
        single.update_elevation(h)
        single.assess_se2(0)
        for m in maps:
            for j0, n in _runs(m.owned_rows()):
                m.update_elevation(np.ascontiguousarray(h[j0:j0 + n]), j0=j0)
        _exchange(maps)
        for m in maps:
            m.assess_se2(0)
        _check_rows(maps, single, J_M, (n_yaw, ny, nx))
        # window shifts (within the pre-generated world patch): own rows of the entered strips, exchange,
        # INCREMENTAL on every rank; the single map FULL
        x, y = robot
        for dx, dy in [(0.93, 0.0), (0.0, -1.27), (-2.05, 3.41)]:
            x, y = x + dx, y + dy
            single.shift_window(x, y)
            I_M, J_M = single.origin()
            h = np.ascontiguousarray(win(I_M, J_M))
            single.update_elevation(h)
            single.assess_se2(0)
            for m in maps:
                di, dj = m.shift_window(x, y)
                assert m.origin() == (I_M, J_M)
                own = set(int(j) for j in m.owned_rows())
                for i0, j0, w, hh in _exposed_strips(di, dj, nx, ny):
                    for a, n in _runs([j for j in range(j0, j0 + hh) if j in own]):
                        m.update_elevation(np.ascontiguousarray(h[a:a + n, i0:i0 + w]), i0=i0, j0=a)
            _exchange(maps)
            for m in maps:
                m.assess_se2(1)
            _check_rows(maps, single, J_M, (n_yaw, ny, nx))
    finally:
        for m in maps + [single]:
            m.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_highres_yaw_slices_equal_single(G):
    from paper_2503_02412_b200 import se2map as S
    cfg = CONFIGS["highres"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    robot = cfg["robot"]
    single = make_map(nx, ny, r, n_yaw, robot=robot)
    maps = [make_map(nx, ny, r, n_yaw, robot=robot, shard_mode=1, rank=g, world_size=G) for g in range(G)]
    try:
        period = single.chain_segments()
        assert all(m.chain_segments() == period for m in maps)
        I_M, J_M = single.origin()
        margin = 30
        world = world_heights(cfg["terrain"], I_M - margin, J_M - margin, nx + 2 * margin, ny + 2 * margin, r)
        H = n_yaw // 2
        for step, (dx, dy) in enumerate([(0.0, 0.0), (0.41, -0.27)]):
            if step:
                x, y = robot[0] + dx, robot[1] + dy
                single.shift_window(x, y)
                for m in maps:
                    m.shift_window(x, y)
                I_M2, J_M2 = single.origin()
            else:
                I_M2, J_M2 = I_M, J_M
            h = np.ascontiguousarray(world[J_M2 - J_M + margin:J_M2 - J_M + margin + ny,
                                           I_M2 - I_M + margin:I_M2 - I_M + margin + nx])
            single.update_elevation(h)
            single.assess_se2(0)
            for m in maps:
                m.update_elevation(h)
                m.assess_se2(1 if step else 0)
            ref = _dev_planes(single, (n_yaw, ny, nx))
            covered = np.zeros(H, bool)
            for g, m in enumerate(maps):
                pl = S.shard_plan(m.params)
                lo, hi = pl["k_lo"], pl["k_hi"]
                assert not covered[lo:hi].any()
                covered[lo:hi] = True
                got = _dev_planes(m, (n_yaw, ny, nx))
                for f in PLANES:
                    for a, b in ((lo, hi), (lo + H, hi + H)):
                        assert _same_bits(got[f][a:b], ref[f][a:b]), (G, g, f, step)
                del got
            assert covered.all()
            del ref
    finally:
        for m in maps + [single]:
            m.close()
        torch.cuda.empty_cache()
