#!/usr/bin/env python
"""Benchmark of the SE(2) traversability hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config large] [--impl ours|reference]

A step = one pass of the whole hot path over the configuration's
map: shift_window (Eq. 4, the robot moves along a path), update_elevation (the full window,
from an HBM-resident world buffer for `value`, from pinned host memory for `e2e`), assess_se2
FULL (Alg. 1 for every SE(2) state), and a batch query of planner states.  Prints ONE JSON line
on rank 0.  Under torchrun (N > 1) every GPU runs its own map of the configuration's size (a batch
of independent maps, one per GPU: weak scaling — the path has no exchange step, so no data-path
collective); value = all ranks' states / the max-over-ranks time.  `--shard rows` instead splits ONE
map across the GPUs in interleaved tile-row bands: each rank is fed only its own rows, the halo rows
its tiles read are exchanged with NCCL send/recv every step (Se2Map.exchange_halo), and it assesses
its own tile rows (strong scaling; SURVEY.md §8(e) "row bands + halo").

`--impl reference`: the FP64 CPU oracle (oracle/, the test reference) timed as it stands on this
host's cores on a bounded random sample of the same workload per step (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.terrain import CONFIGS, DEFAULT_RISK, world_heights  # noqa: E402

METRIC = "SE(2) cells assessed/sec (full local-map update)"
UNIT = "states/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="large", choices=["large", "highres", "paper", "tiny"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--queries", type=int, default=4096)
    ap.add_argument("--shard", default="auto", choices=["auto", "maps", "rows", "yaw"],
                    help="N > 1: 'rows' = ONE map split into interleaved tile-row bands, each rank fed only its own "
                         "rows, halo rows exchanged inside the library by NCCL send/recv every step "
                         "(se2m_exchange_halo); 'yaw' = ONE map, every rank fed the whole window, each assessing "
                         "its slice of yaw bins (both strong scaling, SURVEY.md §8(e)); 'maps' = one independent "
                         "map per GPU (weak scaling); 'auto' (default) = the north_star's split of the config: "
                         "rows for large, yaw for highres, maps otherwise")
    return ap.parse_args()


def stencil_cells(cfg):
    """Mean |P_k| (footprint cells) over yaw bins: for the roofline's per-state work.
    Counted from the oracle-independent rule R5 re-stated here (host arithmetic, no library code)."""
    r, ex, ey, n = cfg["r"], cfg["ex"], cfg["ey"], cfg["n_yaw"]
    a, b = ex / r, ey / r
    R = int(math.ceil(max(a, b))) + 1
    di, dj = np.meshgrid(np.arange(-R, R + 1), np.arange(-R, R + 1))
    tot = 0
    for k in range(n):
        kr = k % (n // 2) if n % 2 == 0 else k
        th = -math.pi + 2 * math.pi * kr / n
        u = di * math.cos(th) + dj * math.sin(th)
        v = -di * math.sin(th) + dj * math.cos(th)
        tot += int(((u / a) ** 2 + (v / b) ** 2 <= 1 + 1e-9).sum())
    return tot / n


def robot_positions(cfg, n):
    """A deterministic back-and-forth path (2-3 cells per step) so the window really shifts."""
    x0, y0 = cfg["robot"]
    r = cfg["r"]
    out = []
    for t in range(n):
        ph = t % 16
        s = ph if ph < 8 else 16 - ph
        out.append((x0 + 0.23 * s + 0.013, y0 + 0.17 * s + 0.011))
    return out, int(math.ceil(0.23 * 8 / r)) + 2


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (pynvml) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)   # ~2 ms: several samples even in a ~25 ms timed region

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def max_over_ranks(vals, world, device=None):
    """Element-wise max over ranks (NCCL on the GPU path, gloo in the CPU tests); identity at N = 1."""
    if world <= 1:
        return list(vals)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def rank_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------------------------------------
def cpu_oracle_rate(cfg, h, budget_s=15.0, seed=0, nthreads=None):
    """The FP64 oracle as it stands, on a bounded uniform random sample of the workload's states."""
    import oracle
    P = oracle.Params(nx=cfg["nx"], ny=cfg["ny"], resolution=cfg["r"], n_yaw=cfg["n_yaw"], ex=cfg["ex"],
                      ey=cfg["ey"], **DEFAULT_RISK)
    nthreads = nthreads or oracle.default_threads()
    rng = np.random.default_rng(seed)
    n, done, t_tot = 20000, 0, 0.0
    while t_tot < budget_s:
        ijk = np.stack([rng.integers(0, cfg["nx"], n), rng.integers(0, cfg["ny"], n),
                        rng.integers(0, cfg["n_yaw"], n)], axis=1).astype(np.int32)
        t0 = time.perf_counter()
        oracle.assess_states(P, h, ijk, nthreads=nthreads)
        dt = time.perf_counter() - t0
        t_tot += dt
        done += n
        n = int(min(max(n * 2, 1), max(20000, done / max(t_tot, 1e-9) * (budget_s - t_tot) + 1)))
    return done / t_tot, done, t_tot, nthreads


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    x, y = cfg["robot"]
    import oracle
    I_M, J_M = oracle.window_origin(x, y, cfg["r"], cfg["nx"], cfg["ny"])
    h = world_heights(cfg["terrain"], I_M, J_M, cfg["nx"], cfg["ny"], cfg["r"])
    # each step a bounded sample: ~6 s, shrunk so that the whole run stays within ~2.5 minutes
    per_step = float(os.environ.get("BENCH_REF_STEP_S", str(max(0.5, min(6.0, 150.0 / max(1, args.steps))))))
    for _ in range(args.warmup):
        cpu_oracle_rate(cfg, h, budget_s=min(1.0, per_step / 4))
    rates, states, secs = [], 0, 0.0
    thr = None
    for s in range(args.steps):
        rate, n, t, thr = cpu_oracle_rate(cfg, h, budget_s=per_step, seed=s + 1)
        rates.append(rate)
        states += n
        secs += t
    value = states / secs
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (T_hills seed 5, SURVEY.md §8(d)); random-init-free: no weights",
            "config": {"workload": args.config, "nx": cfg["nx"], "ny": cfg["ny"], "n_yaw": cfg["n_yaw"],
                       "resolution_m": cfg["r"], "footprint_m": [cfg["ex"], cfg["ey"]]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                             "sample": "per step: uniform random (i,j,k) states of the %s window, ~%.0f s of "
                                       "FP64 oracle work (%d states total)" % (args.config, per_step, states)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
def main():
    args = parse()
    cfg = dict(CONFIGS[args.config])
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2503_02412_b200 import se2map as S

    world, rank, local = rank_env()
    if args.shard == "auto":
        args.shard = {"large": "rows", "highres": "yaw"}.get(args.config, "maps")
    if world > 1:  # NCCL's communicator-init lines (nRanks, transports) on stderr, for the scaling record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    n_states = nx * ny * n_yaw
    K, W = args.steps, max(args.warmup, 3)
    positions, margin = robot_positions(cfg, K + W + 2)
    # multi-GPU: a batch of independent maps, one per GPU (weak scaling: the path needs no exchange,
    # SURVEY.md §8(e) "batches of maps"); rank g's robot drives the same path 1 km further east.
    # --shard rows: one map, every rank on the same path, row bands + NCCL halo exchange (strong scaling)
    rows_mode = args.shard == "rows" and world > 1
    yaw_mode = args.shard == "yaw" and world > 1
    one_map = rows_mode or yaw_mode
    off_x = 0.0 if one_map else 1000.0 * rank
    positions = [(x + off_x, y) for (x, y) in positions]
    robot0 = (cfg["robot"][0] + off_x, cfg["robot"][1])

    shard_kw = dict(shard_mode=S.SE2M_SHARD_ROWS if rows_mode else S.SE2M_SHARD_YAW, rank=rank,
                    world_size=world) if one_map else {}
    nccl_version = None
    if rows_mode:
        # the library's own NCCL communicator carries the halo (se2m_exchange_halo); torch.distributed only
        # bootstraps its unique id (plumbing): rank 0 makes it, a broadcast hands it to the other ranks
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid, nccl_version = S.nccl_unique_id()
            idt.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
        dist.broadcast(idt, src=0)
        shard_kw["nccl_unique_id"] = bytes(idt.cpu().numpy().tobytes())
    m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, ellipse_ex=cfg["ex"], ellipse_ey=cfg["ey"],
                 robot_x=robot0[0], robot_y=robot0[1], device=local, cuda_stream=stream.cuda_stream, **shard_kw)
    I_M0, J_M0 = m.origin()                        # Eq. 4 window origin of the first position
    # world buffer covering every window of the path, resident in HBM (inputs of `value`)
    WX, WY = nx + 2 * margin, ny + 2 * margin
    WI0, WJ0 = I_M0 - margin, J_M0 - margin
    t0 = time.time()
    world_h = world_heights(cfg["terrain"], WI0, WJ0, WX, WY, r)
    gen_s = time.time() - t0
    world_d = torch.from_numpy(world_h).to(dev)
    world_pinned = torch.from_numpy(world_h).pin_memory()

    rng = np.random.default_rng(1)
    l2_flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def window_view(src, I_M, J_M):
        oi, oj = I_M - WI0, J_M - WJ0
        return src[oj:oj + ny, oi:oi + nx]

    def queries(I_M, J_M):
        nq = args.queries
        return np.stack([rng.uniform(I_M * r, (I_M + nx) * r, nq), rng.uniform(J_M * r, (J_M + ny) * r, nq),
                         rng.uniform(-math.pi, math.pi, nq)], axis=1)

    def own_row_runs():
        """(j0, n) runs of the window rows this rank owns (all rows unless --shard rows)."""
        runs = []
        for j in m.owned_rows():
            if runs and runs[-1][0] + runs[-1][1] == j:
                runs[-1][1] += 1
            else:
                runs.append([int(j), 1])
        return runs

    def update(src, I_M, J_M, host=False):
        """H2: the whole window, or (--shard rows) the rank's own rows only, then the halo exchange."""
        v = window_view(src, I_M, J_M)
        if not rows_mode:
            m.update_elevation(v.numpy() if host else v)
            return
        for j0, n in own_row_runs():
            m.update_elevation(v[j0:j0 + n].numpy() if host else v[j0:j0 + n], j0=j0)
        m.exchange_halo()

    def step(t, src):
        m.shift_window(*positions[t])
        I_M, J_M = m.origin()
        update(src, I_M, J_M)
        m.assess_se2(S.SE2M_FULL)
        return I_M, J_M

    # ---- device-resident `value` ----------------------------------------------------------------
    with torch.cuda.stream(stream):
        for t in range(W):
            I_M, J_M = step(t, world_d)
            m.query(queries(I_M, J_M))
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        evk = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        # H10 planner queries of every timed step, prepared up front in pinned memory (states inside the
        # step's window: within nx/2 - 1 cells of the robot), read back asynchronously (se2m_query_async):
        # the host queues step t+1 while the GPU still runs step t, as a pipelined robot loop would
        nq = args.queries
        q_in, q_out = [], []
        TYq = m.tile_info()[1]
        for t in range(K):
            x0, y0 = positions[W + t]
            hx, hy = (nx / 2 - 1) * r, (ny / 2 - 1) * r
            ys = rng.uniform(y0 - hy, y0 + hy, nq)
            if rows_mode:  # a row-band rank answers for its own rows: the planner routes queries by row
                Jq = np.floor(ys / r).astype(np.int64)
                Jq = Jq + (((rank - np.floor_divide(Jq, TYq)) % world) * TYq)   # same offset in the own band
                Jlo = int(math.floor(y0 / r)) - ny // 2
                Jq = np.where(Jq < Jlo + ny, Jq, Jq - world * TYq)
                ys = (Jq + rng.uniform(0.01, 0.99, nq)) * r
            q = np.stack([rng.uniform(x0 - hx, x0 + hx, nq), ys, rng.uniform(-math.pi, math.pi, nq)], axis=1)
            q_in.append(torch.from_numpy(q).pin_memory())
            q_out.append(torch.empty((5, nq), dtype=torch.float32).pin_memory())
        launches0 = m.launch_count()
        with ClockSampler(local) as clk:
            for t in range(K):
                l2_flush.zero_()                    # L2 flush between timed steps (outside the events)
                tt = W + t
                ev[t][0].record(stream)
                m.shift_window(*positions[tt])
                I_M, J_M = m.origin()
                update(world_d, I_M, J_M)
                evk[t][0].record(stream)
                m.assess_se2(S.SE2M_FULL)
                evk[t][1].record(stream)
                m.query_async(q_in[t], q_out[t])     # H10 (D2H of the answers inside the step)
                ev[t][1].record(stream)
            stream.synchronize()
        n_unanswered = sum(int(torch.isnan(o[0]).sum()) for o in q_out)  # all queries lie inside the window
        launches = m.launch_count() - launches0
        step_ms = [a.elapsed_time(b) for a, b in ev]
        kern_ms = [a.elapsed_time(b) for a, b in evk]
    tot_s = sum(step_ms) / 1e3
    kern_s = sum(kern_ms) / 1e3
    tot_s, kern_s = max_over_ranks([tot_s, kern_s], world, dev)
    n_jobs = 1 if one_map else world               # maps assessed per step (rows / yaw: one map split)
    own_states = len(m.owned_rows()) * nx * n_yaw  # this rank's states of the last window
    if yaw_mode:
        pl = S.shard_plan(m.params)
        own_states = (pl["k_hi"] - pl["k_lo"]) * (2 if n_yaw % 2 == 0 else 1) * nx * ny
    value = n_jobs * n_states * K / tot_s          # all ranks' states / the slowest rank's time

    # ---- e2e: public API with host buffers (H2D of the step's map from pinned memory, D2H of the
    #      risk map to pinned memory: the paper sends the risk map back to the CPU) -----
    e2e = None
    if not args.no_e2e:
        # Risk / traversability are pi-periodic in theta (R13 / R23): the planner's copy holds the n_yaw / 2
        # representative planes (se2m_download_compact_rep), filled asynchronously on the library's copy
        # stream, so step t's D2H overlaps step t+1's H2D + assess; the timed region ends after the last
        # D2H completed (host wall clock around the loop, both streams synchronised).
        wpr = (nx + 31) // 32
        n_rep = n_yaw // 2 if n_yaw % 2 == 0 else n_yaw
        own = len(m.owned_rows())                   # row-band ranks download their own rows only
        comp = [{"risk_h": torch.empty((n_rep, own, nx), dtype=torch.float16).pin_memory(),
                 "trav_bits": torch.empty((n_rep, own, wpr), dtype=torch.int32).pin_memory()} for _ in range(2)]
        ke = max(3, min(K, 8))
        with torch.cuda.stream(stream):
            for t in range(2):                      # warm the staging buffers
                m.shift_window(*positions[t])
                I_M, J_M = m.origin()
                update(world_pinned, I_M, J_M, host=True)
                m.assess_se2(S.SE2M_FULL)
                m.download_compact_rep(out=comp[t % 2])
            m.synchronize()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for t in range(ke):
                m.shift_window(*positions[W + t])
                I_M, J_M = m.origin()
                update(world_pinned, I_M, J_M, host=True)
                m.assess_se2(S.SE2M_FULL)
                m.download_compact_rep(out=comp[t % 2])
            m.synchronize()
            e2e_s = time.perf_counter() - t0
        e2e_s = max_over_ranks([e2e_s], world, dev)[0]
        e2e = {"value": n_jobs * n_states * ke / e2e_s, "unit": UNIT, "h2d_bytes_per_step": own * nx * 4,
               "d2h_bytes_per_step": n_rep * own * nx * 2 + n_rep * own * wpr * 4, "ms_per_step": e2e_s / ke * 1e3,
               "steps": ke,
               "note": "per step: H2D of the full window (--shard rows: the rank's own rows, then the NCCL halo "
                       "exchange) from pinned host memory, assess FULL, and D2H of the "
                       "risk map (IEEE binary16: within the north_star risk tolerance of the FP32 state) + traversable bits in logical order to pinned host "
                       "memory (se2m_download_compact_rep: the n_yaw/2 representative planes, Risk being "
                       "pi-periodic in theta; the paper sends the risk map to the CPU, PAPER.md:95); D2H of step "
                       "t overlaps step t+1 on a copy stream; host wall clock to the last D2H"}

    if rank != 0:
        m.close()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (assess_kernel) -----------------------------------------------
    peaks = measured_peaks()
    clocks = clk.summary()
    sm_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = n_sm * 128 * sm_max * 1e6 / 1e12      # FP32-pipe lane-ops/s (FMA = 1 op), Tops/s
    Pk = stencil_cells(cfg)
    W_state = 4 * Pk + 200                           # SURVEY.md §8(d) algorithmic ops per state
    states_per_launch = own_states if one_map else n_states   # per rank
    t_kernel = kern_s / K                            # per launch (update scatter included: < 1%)
    achieved = states_per_launch * W_state / t_kernel / 1e12
    bytes_state = 16.0 + 1.0 / 8.0 + (4.0 + 1.0 / 8.0) / n_yaw
    hbm_gbs = states_per_launch * bytes_state / t_kernel / 1e9
    hbm_peak = peaks.get("hbm_gbs", 6450.6)
    prof = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_ncu_summary.json")))
    except Exception:
        pass
    # The binding roofline is HBM: the write stream of the state records (16 B + 1 bit per state) takes
    # 0.72 ms per large-map launch at the measured copy bandwidth, while the kernel's own FP32-pipe work
    # (ncu: FMA-pipe cycles) fits in less.  The paper-algorithm ALU figure is kept as a
    # secondary, "effective" number: it counts W = 4|P_k| + 200 ops/state that the kernel avoids.
    roofline = {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_gbs / hbm_peak,
                "traffic": prof.get("dram_bytes_per_launch"), "kernel": "assess_kernel",
                "ms_per_launch": t_kernel * 1e3, "bytes_per_state": bytes_state,
                "algorithmic_bytes_per_launch": states_per_launch * bytes_state,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write bytes)",
                "alu": {"achieved": achieved, "peak": alu_peak, "unit": "Tops/s (FP32-pipe ops, FMA=1)",
                        "frac_effective": achieved / alu_peak, "ops_per_state": W_state,
                        "mean_footprint_cells": Pk,
                        "peak_source": "148 SMs x 128 FP32 lanes x sm_max_mhz (B200_PROFILING.md unit counts; "
                                       "FFMA2/FADD measured at 128 lanes/clk/SM in profiles/r01_pipes_microbench.json)",
                        "note": "counts the paper-algorithm work W = 4|P_k| + 200 FP32 ops/state (SURVEY.md §8(d)); "
                                "the kernel computes the same sums with prefix differences and yaw-chain updates and "
                                "shares one eigen-solve between bins k and k + n/2, so this effective fraction exceeds "
                                "1; the kernel's own FP32-pipe use is the ncu fma-pipe percentage below"}}
    if prof:
        roofline["ncu"] = {k: v for k, v in prof.items()
                           if k not in ("dram_bytes_per_launch", "hot_lines", "launch_shares")}
        roofline["ncu"]["source"] = "profiles/latest_ncu_summary.json (ncu --set full of this kernel)"

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        h = world_heights(cfg["terrain"], *m.origin(), nx, ny, r)
        rate, n_done, secs, thr = cpu_oracle_rate(cfg, h, budget_s=float(os.environ.get("BENCH_CPU_S", "15")))
        rate1, n1, secs1, _ = cpu_oracle_rate(cfg, h, budget_s=2.0, seed=1, nthreads=1)
        cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": "oracle",
               "sample": "%d uniform random (i,j,k) states of the %s window (FP64 C oracle, %.1f s)"
                         % (n_done, args.config, secs),
               "single_thread_value": rate1, "cpu_model": cpu_model()}

    extras = {}
    if not args.no_extras and world == 1:
        extras = small_configs(S, stream, torch)
        extras.update(next_rows(m, stream, torch, cfg))
        extras.update(paper_pipeline(S, stream, torch))
        extras.update(highres_update(S, stream, torch))

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": tot_s / K * 1e3, "higher_is_better": True, "scaling": "strong" if one_map else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: T_hills seed 5 (sinusoid hills, slope_rms 0.5, rocks, 1 cm noise; SURVEY.md §8(d)); "
                    "no weights",
            "config": {"workload": args.config, "nx": nx, "ny": ny, "n_yaw": n_yaw, "resolution_m": r,
                       "footprint_m": [cfg["ex"], cfg["ey"]], "states_per_step": n_jobs * n_states,
                       "states_per_gpu_per_step": own_states if one_map else n_states,
                       "parallelism": ("rows%d (one map, interleaved tile-row bands, NCCL halo exchange)" % world
                                       if rows_mode else "yaw%d (one map, yaw slices, replicated input)" % world
                                       if yaw_mode else "batch%d (one independent map per GPU)" % world)
                                      if world > 1 else "single",
                       "l2": "256 MB buffer written between timed steps (outside the step events); "
                             "each step also writes %.2f GB of outputs" % (n_states * 16.125 / 1e9),
                       "step": ("shift_window + update_elevation(own rows, D2D from HBM) + exchange_halo (NCCL) + "
                                "assess_se2(FULL, own tile rows) + query_async(%d states)" if rows_mode else
                                "shift_window + update_elevation(full window, D2D from HBM) + assess_se2(FULL) + "
                                "query_async(%d states, answers D2H to pinned memory)") % args.queries,
                       "queries_unanswered": n_unanswered,
                       "halo_transport": ("se2m_exchange_halo: the library's NCCL communicator (version %s, %d ranks), "
                                          "ncclSend/ncclRecv of the packed halo slabs on the map's stream"
                                          % (nccl_version, world)) if rows_mode else None},
            "ms_per_full_update": kern_s / K * 1e3,
            "ms_per_step_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
            "ms_per_full_update_p10_p50_p90": [float(np.percentile(kern_ms, q)) for q in (10, 50, 90)],
            "gpu_launches": int(launches), "clocks": clocks, "roofline": roofline, "e2e": e2e,
            "cpu_baseline": cpu, "extras": extras,
            "setup": {"terrain_gen_s": round(gen_s, 2)}}
    print(json.dumps(line), flush=True)
    m.close()                                      # free the map's streams / memory before interpreter teardown
    del world_d, l2_flush
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def next_rows(m, stream, torch, cfg, d_max=2.0, n_queries=1 << 20):
    """SURVEY §8(f) rows built so far, on the bench map after its last assess: NEXT-2 SDF of the Risk = 1
    set (all layers, d_max = 2 m) and NEXT-3 trilinear Risk queries with gradients (1 Mi random states)."""
    out = {}
    with torch.cuda.stream(stream):
        m.compute_sdf(d_max)                         # warm
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            m.compute_sdf(d_max)
        e1.record(stream)
        stream.synchronize()
        sdf_ms = e0.elapsed_time(e1) / 5
    layers = cfg["n_yaw"] // 2 if cfg["n_yaw"] % 2 == 0 else cfg["n_yaw"]
    out["sdf_ms"] = sdf_ms
    out["sdf_cells_per_s"] = cfg["nx"] * cfg["ny"] * layers / (sdf_ms * 1e-3)
    out["sdf_d_max_m"] = d_max
    I_M, J_M = m.origin()
    r, nx, ny = cfg["r"], cfg["nx"], cfg["ny"]
    rng = np.random.default_rng(7)
    q = np.stack([rng.uniform((I_M + 1) * r, (I_M + nx - 1) * r, n_queries),
                  rng.uniform((J_M + 1) * r, (J_M + ny - 1) * r, n_queries),
                  rng.uniform(-math.pi, math.pi, n_queries)], axis=1)
    # NEXT-3: warmed at the timed size (staging buffers grown), CUDA events on the map's stream; device-resident
    # queries (kernel throughput) and pinned host buffers (H2D of the queries + kernel + D2H of the answers)
    q_pin = torch.from_numpy(q).pin_memory()
    o_pin = torch.empty((4, n_queries), dtype=torch.float32).pin_memory()
    q_dev = q_pin.to(f"cuda:{torch.cuda.current_device()}")
    o_dev = torch.empty((4, n_queries), dtype=torch.float32, device=q_dev.device)
    res = {}
    with torch.cuda.stream(stream):
        for name, (qi, oi) in (("device", (q_dev, o_dev)), ("host", (q_pin, o_pin))):
            for _ in range(3):
                m.query_trilinear_async(qi, oi, 0)
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                m.query_trilinear_async(qi, oi, 0)
            e1.record(stream)
            stream.synchronize()
            res[name] = n_queries * 10 / (e0.elapsed_time(e1) * 1e-3)
    out["trilinear_queries_per_s"] = res["device"]
    out["trilinear_queries_per_s_host_buffers"] = res["host"]
    out["trilinear_nan_answers"] = int(torch.isnan(o_pin[0]).sum())
    out["trilinear_note"] = ("se2m_query_trilinear_async of 1 Mi random states (Risk field, value + gradient), CUDA "
                             "events over 10 calls after 3 warm-up calls of the same size: device-resident queries "
                             "(kernel) and pinned host buffers (H2D + kernel + D2H)")
    m.inpaint()                                      # NEXT-4 on the bench map (fully known: a pass over
    t0 = time.perf_counter()                         # every cell, nothing to fill)
    for _ in range(5):
        m.inpaint()
    out["inpaint_ms"] = (time.perf_counter() - t0) / 5 * 1e3
    out["inpaint_note"] = "se2m_inpaint on the bench map, host wall clock incl. its counter read-back"
    return out


def highres_update(S, stream, torch, reps=10):
    """BASELINE.json's other large config (800 x 800 @ 0.05 m x 72 bins = 46 M states, footprint radius
    16 cells): device time of one FULL assess, median over reps."""
    cfg = CONFIGS["highres"]
    nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
    m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, ellipse_ex=cfg["ex"], ellipse_ey=cfg["ey"],
                 robot_x=cfg["robot"][0], robot_y=cfg["robot"][1], cuda_stream=stream.cuda_stream)
    h = world_heights(cfg["terrain"], *m.origin(), nx, ny, r)
    with torch.cuda.stream(stream):
        m.update_elevation(h)
        for _ in range(3):
            m.assess_se2(0)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            m.assess_se2(0)
            e1.record(stream)
            ts.append((e0, e1))
        stream.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ts)
    m.close()
    n = nx * ny * n_yaw
    t = ms[len(ms) // 2]
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6450.6)
    bytes_state = 16.0 + 1.0 / 8.0 + (4.0 + 1.0 / 8.0) / n_yaw
    W_state = 4 * stencil_cells(cfg) + 200
    out = {"highres_ms": t, "highres_states": n, "highres_states_per_s": n / (t * 1e-3),
           "highres_W_ops_per_state": W_state}
    # the binding bound of this config is the kernels' own instruction issue, not HBM: its floor is
    # the warp instructions of one assess call (ncu, profiles/) at one instruction per cycle per scheduler
    roof = {"hbm": {"achieved_gbs": n * bytes_state / (t * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                    "frac": n * bytes_state / (t * 1e-3) / 1e9 / hbm_peak, "bytes_per_state": bytes_state}}
    # SURVEY.md §8(d)'s gate (>= 60 % of the FP32 roofline of the paper-algorithm work W per state), "effective"
    # as for the large map: the kernel does fewer operations than W by prefix differences and the yaw chain
    sm_mhz = peaks.get("sm_max_mhz") or 1965.0
    n_sm_dev = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    alu_peak = n_sm_dev * 128 * sm_mhz * 1e6 / 1e12
    alu = n * W_state / (t * 1e-3) / 1e12
    roof["alu"] = {"achieved": alu, "peak": alu_peak, "unit": "Tops/s (FP32-pipe ops, FMA=1)",
                   "frac_effective": alu / alu_peak, "ops_per_state": W_state}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_ncu_highres.json")))
        n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        mhz = prof.get("sm_frequency_ghz", 1.9) * 1e3
        floor_ms = prof["executed_instructions_per_call"] / (4 * n_sm * mhz * 1e6) * 1e3
        roof["issue"] = {"floor_ms": floor_ms, "frac": floor_ms / t, "executed_warp_instructions_per_call":
                         prof["executed_instructions_per_call"], "sm_mhz": mhz,
                         "source": "profiles/latest_ncu_highres.json (ncu --set full of one assess call: both kernels)"}
        roof["bound"] = "issue"
    except Exception:
        roof["bound"] = "issue (no ncu summary in profiles/)"
    out["highres_roofline"] = roof
    return out


def paper_pipeline(S, stream, torch, n_frames=6, n_iters=40, warm=4):
    """The paper's own headline point: the WHOLE local-mapping update at
    972,000 SE(2) states (180 x 180 cells at 0.1 m x 30 yaw bins) in < 50 ms.  Per LiDAR frame (16 beams x
    1800 azimuths, synth/lidar.py, host arrays): shift_window (Eq. 4) + integrate_scan (NEXT-1: filter,
    variance, ray casting, KF; synchronises) + assess_se2 FULL over all 972,000 states of the
    nearest-neighbour inpainted map (NEXT-4, params.inpaint = 1, as in the paper's timing: P:248);
    host wall clock per frame, inputs from host memory.  n_frames scans along a path are replayed
    back and forth (ping-pong) for n_iters frames (scan synthesis is slow on the host)."""
    from synth.lidar import scan
    from synth.terrain import Hills
    terrain = Hills(seed=31)
    nx = ny = 180
    r, n_yaw = 0.1, 30
    path = [(0.37 + 0.15 * t, 0.61 + 0.05 * t, 0.3 + 0.02 * t) for t in range(n_frames)]
    frames = [scan(terrain, x, y, yaw, seed=500 + t, n_az=1800) for t, (x, y, yaw) in enumerate(path)]
    cyc = list(range(n_frames)) + list(range(n_frames - 2, 0, -1))
    m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, robot_x=path[0][0], robot_y=path[0][1],
                 cuda_stream=stream.cuda_stream, inpaint=1)
    ts, tf, npts = [], [], []
    for it in range(n_iters):
        f = cyc[it % len(cyc)]
        (x, y, _), fr = path[f], frames[f]
        pose = S.Pose.from_arrays(fr.R_B, fr.p_B, fr.R_BS, fr.p_BS, fr.Sigma_S, fr.Sigma_R, fr.Sigma_B)
        stream.synchronize()
        t0 = time.perf_counter()
        m.shift_window(x, y)
        m.integrate_scan(fr.points_s, pose)          # synchronises (reads its counters)
        t1 = time.perf_counter()
        m.assess_se2(0)                              # (inpaints first: the map changed)
        stream.synchronize()
        if it >= warm:
            ts.append(time.perf_counter() - t0)
            tf.append(t1 - t0)
            npts.append(len(fr.points_s))
    m.close()
    ms = sorted(1e3 * v for v in ts)
    return {"paper_pipeline_ms_median": statistics.median(ms), "paper_pipeline_ms_p90": ms[int(0.9 * (len(ms) - 1))],
            "paper_pipeline_frontend_ms_median": 1e3 * statistics.median(tf),
            "paper_pipeline_states": nx * ny * n_yaw, "paper_pipeline_points_per_frame": int(np.mean(npts)),
            "paper_pipeline_frames": len(ms),
            "paper_pipeline_note": "whole mapping update per LiDAR frame (shift + integrate_scan + NN "
                                   "inpainting + FULL assess of 180x180x30 states), host wall clock, host "
                                   "inputs; the paper: < 50 ms on a GTX-1660-class GPU (P:248-250)"}


def exposed_strips(di, dj, nx, ny):
    """Window-local rectangles (i0, j0, w, h) that entered the window after a shift by (di, dj)."""
    if abs(di) >= nx or abs(dj) >= ny:
        return [(0, 0, nx, ny)]
    rects = []
    if di > 0:
        rects.append((nx - di, 0, di, ny))
    elif di < 0:
        rects.append((0, 0, -di, ny))
    if dj > 0:
        rects.append((0, ny - dj, nx, dj))
    elif dj < 0:
        rects.append((0, 0, nx, -dj))
    return rects


def small_configs(S, stream, torch):
    """paper-like FULL update time and the rolling-window stream step (INCREMENTAL), in microseconds."""
    out = {}
    from synth.terrain import robot_path
    for name in ("paper", "stream"):
        cfg = CONFIGS[name]
        nx, ny, r, n_yaw = cfg["nx"], cfg["ny"], cfg["r"], cfg["n_yaw"]
        m = S.Se2Map(nx=nx, ny=ny, n_yaw=n_yaw, resolution=r, ellipse_ex=cfg["ex"], ellipse_ey=cfg["ey"],
                     robot_x=cfg["robot"][0], robot_y=cfg["robot"][1], cuda_stream=stream.cuda_stream)
        I_M, J_M = m.origin()
        h = world_heights(cfg["terrain"], I_M, J_M, nx, ny, r)
        with torch.cuda.stream(stream):
            hd = torch.from_numpy(h).cuda()
            m.update_elevation(hd)
            if name == "paper":
                for _ in range(10):
                    m.assess_se2(0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(100):
                    m.assess_se2(0)
                e1.record(stream)
                stream.synchronize()
                out["paper_full_us"] = e0.elapsed_time(e1) * 10.0
                out["paper_states"] = nx * ny * n_yaw
            else:
                path = robot_path(cfg["path_seed"], cfg["n_steps"] + 20, r, *cfg["robot"])  # 20 warm + 1000 timed
                # strips come from a pre-generated world patch covering the path
                xs, ys = path[:, 0], path[:, 1]
                I0 = int(math.floor(xs.min() / r)) - nx // 2 - 2
                J0 = int(math.floor(ys.min() / r)) - ny // 2 - 2
                Wd = int(math.ceil((xs.max() - xs.min()) / r)) + nx + 6
                Hd = int(math.ceil((ys.max() - ys.min()) / r)) + ny + 6
                wh = torch.from_numpy(world_heights(cfg["terrain"], I0, J0, Wd, Hd, r)).cuda()
                m.assess_se2(0)
                ts = []
                warm = 20                            # first steps: allocations / first-launch setup
                for t in range(1, len(path)):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    # H1 + H2 + H9 in one call (se2m_step): recentre, fill the entered cells from the
                    # device-resident world patch, INCREMENTAL assess
                    m.step(*path[t], wh, I0, J0)
                    e1.record(stream)
                    if t > warm:
                        ts.append((e0, e1))
                stream.synchronize()
                us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
                out["stream_us_per_step_mean"] = sum(us) / len(us)
                out["stream_us_per_step_p99"] = us[int(0.99 * (len(us) - 1))]
                out["stream_steps"] = len(us)
        m.close()
    return out


if __name__ == "__main__":
    main()
