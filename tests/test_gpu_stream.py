"""Rolling-window stream (BASELINE.json config 3) and sharded maps on one GPU.

* Q13: INCREMENTAL after any sequence of shifts == FULL on the same map, bit-exact, every step checked.
* Parity with the oracle at steps 1, 10, 100, 1000 (SURVEY.md §8(d) 'stream').
* Sharded (yaw slices / row bands) == unsharded, bit-exact, with the ranks emulated as independent
  handles on one GPU (no rank waits on another, so this is safe on a single device).
"""
import numpy as np
import pytest

import oracle
from synth.terrain import CONFIGS, robot_path, world_heights
from tests.gpu_common import make_map, oracle_params
from tests.parity import compare

pytestmark = pytest.mark.gpu


def _exposed_strips(di, dj, nx, ny):
    """Window-local rectangles (i0, j0, w, h) that entered the window after a shift by (di, dj)."""
    rects = []
    if abs(di) >= nx or abs(dj) >= ny:
        return [(0, 0, nx, ny)]
    if di > 0:
        rects.append((nx - di, 0, di, ny))
    elif di < 0:
        rects.append((0, 0, -di, ny))
    if dj > 0:
        rects.append((0, ny - dj, nx, dj))
    elif dj < 0:
        rects.append((0, 0, nx, -dj))
    return rects


def _equal(a, b):
    return all(np.array_equal(a[f], b[f], equal_nan=True) for f in a)


def test_stream_incremental_equals_full_and_oracle():
    cfg = CONFIGS["stream"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    path = robot_path(cfg["path_seed"], cfg["n_steps"], r, *cfg["robot"])
    inc = make_map(nx, ny, r, n_yaw, robot=tuple(path[0]))
    full = make_map(nx, ny, r, n_yaw, robot=tuple(path[0]))
    I_M, J_M = inc.origin()
    h0 = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
    for m in (inc, full):
        m.update_elevation(h0)
        m.assess_se2(0)
    checkpoints = {1, 10, 100, 1000}
    n_shifts = 0
    for t in range(1, len(path)):
        x, y = path[t]
        d1 = inc.shift_window(x, y)
        d2 = full.shift_window(x, y)
        assert d1 == d2
        n_shifts += d1 != (0, 0)
        I_M, J_M = inc.origin()
        assert (I_M, J_M) == oracle.window_origin(x, y, r, nx, ny)
        for (i0, j0, w, h) in _exposed_strips(*d1, nx, ny):
            strip = world_heights(cfg["terrain"], I_M + i0, J_M + j0, w, h, r)
            inc.update_elevation(strip, i0=i0, j0=j0)
            full.update_elevation(strip, i0=i0, j0=j0)
        inc.assess_se2(1)
        full.assess_se2(0)
        if t % 25 == 0 or t in checkpoints:
            gi, gf = inc.download(), full.download()
            assert _equal(gi, gf), "INCREMENTAL != FULL at step %d" % t
            if t in checkpoints:
                h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
                orc = oracle.assess_all(oracle_params(nx, ny, r, n_yaw), h)
                rep = compare(gi, orc)
                print("step", t, rep)
                assert rep["ok"], (t, rep)
    assert n_shifts > 300


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("G", [2, 3])
def test_sharded_equals_single(mode, G):
    cfg = dict(CONFIGS["paper"])
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    single = make_map(nx, ny, r, n_yaw, robot=cfg["robot"])
    I_M, J_M = single.origin()
    h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
    single.update_elevation(h)
    single.assess_se2(0)
    ref = single.download()
    merged = {f: np.full_like(v, np.nan if v.dtype != np.uint8 else 0) for f, v in ref.items()}
    for rank in range(G):
        m = make_map(nx, ny, r, n_yaw, robot=cfg["robot"], shard_mode=mode, rank=rank, world_size=G)
        m.update_elevation(h)
        m.assess_se2(0)
        g = m.download()
        if mode == 1:
            from paper_2503_02412_b200 import se2map as S
            plan = S.shard_plan(m.params)
            H, lo, hi = plan["n_rep"], plan["k_lo"], plan["k_hi"]
            own = np.zeros(n_yaw, bool)
            own[lo:hi] = True
            own[lo + H:hi + H] = True
            mask = np.broadcast_to(own[:, None, None], ref["risk"].shape)
        else:
            J = np.arange(J_M, J_M + ny)
            TY = m.tile_info()[1]
            own_rows = (np.floor_divide(J, TY) % G) == rank
            mask = np.broadcast_to(own_rows[None, :, None], ref["risk"].shape)
        for f in merged:
            merged[f][mask] = g[f][mask]
        # states the rank does not own come back as NaN / 0 (downloads never expose stale records)
        assert np.all(np.isnan(g["risk"][~mask])) and np.all(g["trav"][~mask] == 0)
        c = m.download_compact()
        assert np.all(c["risk_h"][~mask] == 1.0)
        if mode == 2:  # the planner copy of a row-band rank: its own rows only, packed
            rows = m.owned_rows()
            assert np.array_equal(rows, np.nonzero(own_rows)[0])
            rep_ = m.download_compact_rep()
            m.synchronize()
            H2 = n_yaw // 2
            assert rep_["risk_h"].shape == (H2, len(rows), nx)
            assert np.array_equal(rep_["risk_h"], c["risk_h"][:H2][:, rows, :])
            assert np.array_equal(rep_["trav_bits"], c["trav_bits"][:H2][:, rows, :])
    assert _equal(merged, ref)


@pytest.mark.parametrize("n_yaw", [72, 36])
def test_chain_map_incremental_and_sharded(n_yaw):
    """A map big enough for the yaw chain: INCREMENTAL after shifts == FULL bit-exact, and yaw / row
    sharding == single, bit-exact (yaw shards replay the chain from the period's restart)."""
    from paper_2503_02412_b200 import se2map as S
    nx, ny, r = 544, 520, 0.1
    terrain = CONFIGS["large"]["terrain"]
    robot = (3.37, -2.61)
    single = make_map(nx, ny, r, n_yaw, robot=robot)
    full = make_map(nx, ny, r, n_yaw, robot=robot)
    I_M, J_M = single.origin()
    h = world_heights(terrain, I_M, J_M, nx, ny, r)
    for m in (single, full):
        m.update_elevation(h)
        m.assess_se2(0)
    for (x, y) in [(3.61, -2.47), (4.02, -2.55), (3.1, -3.3), (3.1, -3.3), (2.2, -1.05)]:
        d = single.shift_window(x, y)
        assert full.shift_window(x, y) == d
        I_M, J_M = single.origin()
        for (i0, j0, w, hh) in _exposed_strips(*d, nx, ny):
            strip = world_heights(terrain, I_M + i0, J_M + j0, w, hh, r)
            single.update_elevation(strip, i0=i0, j0=j0)
            full.update_elevation(strip, i0=i0, j0=j0)
        single.assess_se2(1)
        full.assess_se2(0)
        assert _equal(single.download(), full.download())
    ref = full.download()
    h = world_heights(terrain, I_M, J_M, nx, ny, r)
    rng = np.random.default_rng(4)
    ijk = np.stack([rng.integers(0, nx, 20000), rng.integers(0, ny, 20000), rng.integers(0, n_yaw, 20000)], 1)
    orc = oracle.assess_states(oracle_params(nx, ny, r, n_yaw), h, ijk.astype(np.int32))
    for mode in (1, 2):
        for G in (2, 3, 5, 8):
            merged = {f: np.full_like(v, np.nan if v.dtype != np.uint8 else 0) for f, v in ref.items()}
            periods = set()
            for rank in range(G):
                m = make_map(nx, ny, r, n_yaw, robot=(2.2, -1.05), shard_mode=mode, rank=rank, world_size=G)
                periods.add(m.chain_segments())
                m.update_elevation(h)
                m.assess_se2(0)
                g = m.download()
                plan = S.shard_plan(m.params)
                if mode == 1:
                    H, lo, hi = plan["n_rep"], plan["k_lo"], plan["k_hi"]
                    own = np.zeros(n_yaw, bool)
                    own[lo:hi] = True
                    own[lo + H:hi + H] = True
                    mask = np.broadcast_to(own[:, None, None], ref["risk"].shape)
                else:
                    J = np.arange(J_M, J_M + ny)
                    mask = np.broadcast_to(((np.floor_divide(J, plan["tile_y"]) % G) == rank)[None, :, None],
                                           ref["risk"].shape)
                for f in merged:
                    merged[f][mask] = g[f][mask]
            # sharding never changes the chain period: a yaw shard starting inside a period replays the
            # chain from its restart, so the merged shards equal the single map bit for bit (pin Q13)
            assert periods == {single.chain_segments()}
            assert _equal(merged, ref), (mode, G)
    # and parity with the oracle on the sample
    rep = compare({f: ref[f][ijk[:, 2], ijk[:, 1], ijk[:, 0]] for f in ref}, orc)
    assert rep["ok"], rep


@pytest.mark.parametrize("step_graph", [0, 1])
def test_step_equals_separate_calls(step_graph):
    """se2m_step (recentre + fill the entered cells from a device world plane + INCREMENTAL) gives the
    same state records, bit for bit, as shift_window + update_elevation(strips) + assess(INCREMENTAL),
    including cells outside the world plane (unknown) and a jump larger than the window."""
    import torch
    cfg = CONFIGS["stream"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    terrain = cfg["terrain"]
    a = make_map(nx, ny, r, n_yaw, robot=cfg["robot"])
    b = make_map(nx, ny, r, n_yaw, robot=cfg["robot"], step_graph=step_graph)  # 1: the step as one CUDA graph
    I0, J0 = a.origin()
    WI0, WJ0, WW, WH = I0 - 40, J0 - 30, nx + 90, ny + 60          # world plane (partly smaller than the path)
    world = world_heights(terrain, WI0, WJ0, WW, WH, r)
    wt = torch.from_numpy(world).cuda()
    h = world_heights(terrain, I0, J0, nx, ny, r)
    for m in (a, b):
        m.update_elevation(h)
        m.assess_se2(0)
    path = [(0.61, 0.77), (1.13, 0.52), (1.13, 0.52), (4.9, 2.3), (-0.4, -1.7), (30.0, 10.0), (0.5, 0.5)]
    for (x, y) in path:
        d = a.shift_window(x, y)
        I_M, J_M = a.origin()
        for (i0, j0, w, hh) in _exposed_strips(*d, nx, ny):
            strip = np.full((hh, w), np.nan, np.float32)
            ii = np.arange(I_M + i0, I_M + i0 + w) - WI0
            jj = np.arange(J_M + j0, J_M + j0 + hh) - WJ0
            oki, okj = (ii >= 0) & (ii < WW), (jj >= 0) & (jj < WH)
            strip[np.ix_(okj, oki)] = world[np.ix_(jj[okj], ii[oki])]
            a.update_elevation(strip, i0=i0, j0=j0)
        a.assess_se2(1)
        assert b.step(x, y, wt, WI0, WJ0) == d
        assert b.origin() == (I_M, J_M)
        assert _equal(a.download(), b.download()), (x, y)
