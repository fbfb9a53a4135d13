"""Row-band sharding with a halo exchange (SURVEY.md §8(e) "row bands + halo"; se2m_halo_* in
include/se2map.h), on one GPU: the G ranks are independent handles, each given ONLY its own rows of the
elevation window (se2m_owned_rows); the halo slabs each rank packs are handed to its neighbours' handles
(the device copy stands in for the NCCL send / recv — no rank waits on another, so this is safe on a
single device).  After the exchange every rank's owned states must equal the unsharded map's, bit-exact,
through FULL and, after window shifts, INCREMENTAL assessment.
"""
import numpy as np
import pytest
import torch

from synth.terrain import CONFIGS, world_heights
from tests.gpu_common import make_map
from tests.test_gpu_stream import _exposed_strips

pytestmark = pytest.mark.gpu


def _runs(rows):
    """Consecutive runs (start, length) of sorted row indices."""
    out = []
    for j in rows:
        if out and out[-1][0] + out[-1][1] == j:
            out[-1][1] += 1
        else:
            out.append([int(j), 1])
    return out


def _update_own_rows(m, h):
    for j0, n in _runs(m.owned_rows()):
        m.update_elevation(np.ascontiguousarray(h[j0:j0 + n]), j0=j0)


def _exchange(maps):
    """The transfer step of Se2Map.exchange_halo with device copies in place of NCCL send / recv."""
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
        m.halo_unpack(to_lo[(g + 1) % G], +1)   # rank g + 1 sent its first rows toward g
        m.halo_unpack(to_hi[(g - 1) % G], -1)   # rank g - 1 sent its last rows toward g
        m.synchronize()


def _merged_owned(maps, ref, J_M, ny):
    merged = {f: np.full_like(v, np.nan if v.dtype != np.uint8 else 0) for f, v in ref.items()}
    G = len(maps)
    for g, m in enumerate(maps):
        TY = m.tile_info()[1]
        own = (np.floor_divide(np.arange(J_M, J_M + ny), TY) % G) == g
        d = m.download()
        for f in merged:
            merged[f][:, own, :] = d[f][:, own, :]
    return merged


def _equal(a, b):
    return all(np.array_equal(a[f], b[f], equal_nan=True) for f in a)


@pytest.mark.parametrize("G", [2, 3, 4])
def test_row_bands_with_halo_exchange_equal_single(G):
    nx, ny, r, n_yaw = 544, 520, 0.1, 36
    terrain = CONFIGS["large"]["terrain"]
    robot = (3.37, -2.61)
    single = make_map(nx, ny, r, n_yaw, robot=robot)
    maps = [make_map(nx, ny, r, n_yaw, robot=robot, shard_mode=2, rank=g, world_size=G) for g in range(G)]
    I_M, J_M = single.origin()
    h = world_heights(terrain, I_M, J_M, nx, ny, r)
    single.update_elevation(h)
    single.assess_se2(0)
    for m in maps:
        _update_own_rows(m, h)
    _exchange(maps)
    for m in maps:
        m.assess_se2(0)
    assert _equal(_merged_owned(maps, single.download(), J_M, ny), single.download())

    # a few window shifts: every rank refills its own rows of the entered strips, exchanges, INCREMENTAL
    for t, (dx, dy) in enumerate([(0.93, 0.0), (0.0, -1.27), (-2.05, 3.41)]):
        x, y = robot[0] + dx, robot[1] + dy
        robot = (x, y)
        single.shift_window(x, y)
        I_M, J_M = single.origin()
        h = world_heights(terrain, I_M, J_M, nx, ny, r)
        single.update_elevation(h)
        single.assess_se2(0)
        for m in maps:
            di, dj = m.shift_window(x, y)
            assert m.origin() == (I_M, J_M)
            own = set(int(j) for j in m.owned_rows())
            for i0, j0, w, hh in _exposed_strips(di, dj, nx, ny):   # entered cells of the rank's own rows
                for a, n in _runs([j for j in range(j0, j0 + hh) if j in own]):
                    m.update_elevation(np.ascontiguousarray(h[a:a + n, i0:i0 + w]), i0=i0, j0=a)
        _exchange(maps)
        for m in maps:
            m.assess_se2(1)
        assert _equal(_merged_owned(maps, single.download(), J_M, ny), single.download()), t


def test_halo_without_exchange_differs():
    """Control: a row-band rank that got only its own rows and NO halo differs near its band edges (so the
    test above really exercises the exchange)."""
    nx, ny, r, n_yaw = 256, 200, 0.1, 8
    terrain = CONFIGS["large"]["terrain"]
    single = make_map(nx, ny, r, n_yaw)
    m = make_map(nx, ny, r, n_yaw, shard_mode=2, rank=0, world_size=2)
    I_M, J_M = single.origin()
    h = world_heights(terrain, I_M, J_M, nx, ny, r)
    single.update_elevation(h)
    single.assess_se2(0)
    _update_own_rows(m, h)
    m.assess_se2(0)
    ref = single.download()
    own = m.owned_rows()
    assert not np.array_equal(m.download()["risk"][:, own], ref["risk"][:, own], equal_nan=True)


def test_halo_api_errors():
    from paper_2503_02412_b200 import se2map as S
    m = make_map(64, 64, 0.1, 8)                                  # unsharded: no halo
    with pytest.raises(S.Se2mError):
        m.halo_size()
    g = make_map(64, 64, 0.1, 8, shard_mode=2, rank=0, world_size=2)
    cap, rows = g.halo_size()
    buf = torch.empty((cap, rows, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(S.Se2mError):
        g.halo_pack(0, buf)                                        # dir must be -1 / +1
    with pytest.raises(S.Se2mError):
        g.halo_unpack(buf, 2)                                      # from must be -1 / +1
