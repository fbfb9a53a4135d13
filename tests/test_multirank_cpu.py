"""CPU, world_size 2 with gloo: the host side of the multi-GPU path (no GPU needed).

* se2m_shard_plan (host-only C ABI call): the ranks' shares partition the representative yaw bins
  (SE2M_SHARD_YAW) and the world tile rows (SE2M_SHARD_ROWS) exactly — disjoint and covering;
* bench.max_over_ranks: the max-over-ranks timing reduction bench.py uses, over gloo.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_02412_b200 import se2map as S
        import bench
        out = {}
        for name, kw in (("large", dict(nx=2000, ny=2000, n_yaw=72, resolution=0.1)),
                         ("highres", dict(nx=800, ny=800, n_yaw=72, resolution=0.05)),
                         ("odd", dict(nx=37, ny=23, n_yaw=5, resolution=0.1))):
            for mode in (S.SE2M_SHARD_YAW, S.SE2M_SHARD_ROWS):
                p = S.default_params(shard_mode=mode, rank=rank, world_size=world, **kw)
                out[(name, mode)] = S.shard_plan(p)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        assert bench.rank_env()[:2] == (world, rank)
        t = bench.max_over_ranks([1.0 + rank, 10.0 - rank], world)
        q.put((rank, gathered, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shard_plan_partitions_and_max_reduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=120) for _ in procs]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    for rank, gathered, t in res:
        assert t == [float(world), 10.0]                     # element-wise max over ranks
        plans = gathered
        for key in plans[0]:
            name, mode = key
            ps = [plans[r][key] for r in range(world)]
            n_rep = ps[0]["n_rep"]
            if mode == 1:                                     # yaw: contiguous, disjoint, covering
                owned = sorted(k for pl in ps for k in range(pl["k_lo"], pl["k_hi"]))
                assert owned == list(range(n_rep)), (key, ps)
                assert all(pl["row_mod"] == 1 for pl in ps)
            else:                                             # rows: TJ mod G == rank, all bins
                assert sorted(pl["row_rank"] for pl in ps) == list(range(world))
                assert all(pl["row_mod"] == world and (pl["k_lo"], pl["k_hi"]) == (0, n_rep) for pl in ps)
                for TJ in range(-7, 40):
                    owners = [r for r, pl in enumerate(ps) if TJ % pl["row_mod"] == pl["row_rank"]]
                    assert len(owners) == 1


def halo_transfer(send_dn, send_up, recv_up, recv_dn, rank: int, world: int):
    """The transfer step of se2m_exchange_halo (csrc/se2map.cu) in the same issue order, over gloo: send_dn ->
    rank - 1, recv_up <- rank + 1 (its send_dn), send_up -> rank + 1, recv_dn <- rank - 1 (its send_up).  With two
    ranks both neighbours are one peer; point-to-point messages between a pair match in issue order, so each
    receive still gets the right slab set (the library's ncclGroupStart/Send/Recv/GroupEnd relies on the same)."""
    lo, hi = (rank - 1) % world, (rank + 1) % world
    ops = [dist.P2POp(dist.isend, send_dn, lo), dist.P2POp(dist.irecv, recv_up, hi),
           dist.P2POp(dist.isend, send_up, hi), dist.P2POp(dist.irecv, recv_dn, lo)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def _halo_worker(rank, world, port, q):
    """Each rank holds only its own rows of a random map; slabs are cut by the library's host-only slab
    plan (se2m_halo_plan), exchanged by halo_transfer (the library's send / recv order) over gloo, and written
    back by the plan of
    the sending rank — then every row the rank's tiles read (owned tile rows +- R_T) must be present."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import torch
        from paper_2503_02412_b200 import se2map as S
        checked = 0
        for nx, ny, r, J_M in ((96, 200, 0.1, 12345), (64, 131, 0.1, -77), (48, 100, 0.05, 3)):
            p = S.default_params(nx=nx, ny=ny, n_yaw=8, resolution=r, shard_mode=S.SE2M_SHARD_ROWS, rank=rank,
                                 world_size=world)
            TY = S.shard_plan(p)["tile_y"]
            truth = np.random.default_rng(J_M & 0xffff).standard_normal((ny, nx)).astype(np.float32)
            J = np.arange(J_M, J_M + ny)
            own = (np.floor_divide(J, TY) % world) == rank
            local = np.full_like(truth, np.nan)
            local[own] = truth[own]

            def pack(sender, last):
                pl = S.halo_plan(p, J_M, sender, last)
                buf = np.full((pl["cap"], pl["slab_rows"], nx), np.nan, np.float32)
                for qi, w0 in enumerate(pl["first_rows"]):
                    for rr in range(pl["slab_rows"]):
                        if w0 is not None and 0 <= w0 + rr - J_M < ny:
                            buf[qi, rr] = local[w0 + rr - J_M]
                return torch.from_numpy(buf)

            def unpack(buf, sender, last):
                pl = S.halo_plan(p, J_M, sender, last)
                for qi, w0 in enumerate(pl["first_rows"]):
                    for rr in range(pl["slab_rows"]):
                        if w0 is not None and 0 <= w0 + rr - J_M < ny:
                            local[w0 + rr - J_M] = buf[qi, rr].numpy()

            send_dn, send_up = pack(rank, 0), pack(rank, 1)
            recv_up, recv_dn = torch.empty_like(send_dn), torch.empty_like(send_up)
            halo_transfer(send_dn, send_up, recv_up, recv_dn, rank, world)
            unpack(recv_up, (rank + 1) % world, 0)
            unpack(recv_dn, (rank - 1) % world, 1)
            R_T = S.halo_plan(p, J_M, rank, 0)["slab_rows"]
            for TJ in np.unique(np.floor_divide(J, TY)):
                if TJ % world != rank:
                    continue
                j0, j1 = max(0, TJ * TY - R_T - J_M), min(ny, TJ * TY + TY + R_T - J_M)
                assert np.array_equal(local[j0:j1], truth[j0:j1]), (nx, ny, J_M, TJ)
                checked += 1
        q.put((rank, checked))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=180) for _ in procs]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert all(n > 0 for _, n in res)


def test_nccl_unique_id_host_only():
    """se2m_nccl_unique_id loads NCCL through the library (dlopen, no GPU) and returns a 128-byte id."""
    from paper_2503_02412_b200 import se2map as S
    a, ver = S.nccl_unique_id()
    b, _ = S.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
    assert ver >= 21800
