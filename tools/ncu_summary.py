#!/usr/bin/env python
"""Summarise an ncu report of the assess kernel into JSON (+ a hot-line / opcode table on stdout).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv] [--out profiles/x.json]

Reads with the local ncu CLI (`--page details/raw/source --csv`); no GPU needed.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    """{kernel ID: ({(section, metric): (value, unit)}, kernel name)} of every captured kernel."""
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    d = {}
    for r in rows[1:]:
        x = dict(zip(h, r))
        kid = x.get("ID", "0")
        m, _ = d.setdefault(kid, ({}, x.get("Kernel Name", "")))
        m[(x.get("Section Name", ""), x.get("Metric Name", ""))] = (x.get("Metric Value", ""), x.get("Metric Unit", ""))
    return d


def raw(rep, names):
    """[{metric: (value, unit)}] per captured kernel, in capture order."""
    rows = ncu_csv(rep, "--page", "raw")
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        out = {}
        for n in names:
            if n in h:
                i = h.index(n)
                out[n] = (vals[i], units[i])
        res.append(out)
    return res


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except Exception:
        return None


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            h = rows[i]
            body = rows[i + 1:]
            break
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in body:
        if len(r) > iV:
            agg[r[iN].split("(")[0]].append(num(r[iV]))
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "total_us": sum(v) / 1e3, "share": sum(v) / tot} for k, v in
            sorted(agg.items(), key=lambda kv: -sum(kv[1]))}


def hot_lines(rep, top=25):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "cuda,sass")
    agg, stall, src = collections.Counter(), collections.Counter(), {}
    for r in rows[3:]:
        if len(r) > 8 and r[2] == "-":
            try:
                agg[int(r[0])] += int(r[7])
                stall[int(r[0])] += int(r[4] or 0)
                src[int(r[0])] = r[1][:100]
            except ValueError:
                pass
    tot, st = max(1, sum(agg.values())), max(1, sum(stall.values()))
    return [(round(e / tot * 100, 2), round(stall[ln] / st * 100, 2), ln, src[ln]) for ln, e in agg.most_common(top)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--launches")
    ap.add_argument("--out")
    a = ap.parse_args()
    dk = details(a.rep)
    # one assess call may be two kernels (the main grid and the vertical-window-edge tiles, <R_T, 1>):
    # the per-kernel fields describe the main one (the longest), the byte / time totals cover the call
    def dur_ms(m):
        v, u = m.get(("GPU Speed Of Light Throughput", "Duration"), ("", ""))
        sc = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
        return num(v) * sc[u] if num(v) is not None and u in sc else 0.0
    ids = sorted(dk, key=lambda k: -dur_ms(dk[k][0]))
    d = dk[ids[0]][0]
    pick = {
        "duration_ms": ("GPU Speed Of Light Throughput", "Duration"),
        "sm_throughput_pct": ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
        "dram_throughput_pct": ("GPU Speed Of Light Throughput", "DRAM Throughput"),
        "l1tex_throughput_pct": ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
        "issue_slots_busy_pct": ("Compute Workload Analysis", "Issue Slots Busy"),
        "ipc_active": ("Compute Workload Analysis", "Executed Ipc Active"),
        "achieved_occupancy_pct": ("Occupancy", "Achieved Occupancy"),
        "registers_per_thread": ("Launch Statistics", "Registers Per Thread"),
        "executed_instructions": ("Instruction Statistics", "Executed Instructions"),
        "sm_frequency_ghz": ("GPU Speed Of Light Throughput", "SM Frequency"),
    }
    s = {k: num(d.get(v, ("", ""))[0]) for k, v in pick.items()}
    dur, unit = d.get(pick["duration_ms"], ("", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
    if num(dur) is not None and unit in scale:  # ncu prints the unit it chose (us or ms)
        s["duration_ms"] = num(dur) * scale[unit]
    rws = raw(a.rep, ["dram__bytes_read.sum", "dram__bytes_write.sum",
                     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                     "smsp__issue_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum",
                     "sm__inst_executed_pipe_xu.sum", "sm__inst_executed_pipe_lsu.sum",
                     "sm__sass_inst_executed_op_shared_ld.sum"])
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def vals(rw):
        o = {}
        for k, (v, u) in rw.items():
            x = num(v)
            if x is not None and u in units:
                x *= units[u]
            o[k] = x
        return o
    per = [vals(rw) for rw in rws]
    order = sorted(dk)                      # raw rows follow the capture order of the IDs
    main_row = order.index(ids[0]) if ids[0] in order else 0
    s.update(per[main_row])
    tot = 0.0
    for v in per:
        if v.get("dram__bytes_read.sum") is not None and v.get("dram__bytes_write.sum") is not None:
            tot += v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
    s["dram_bytes_per_launch"] = tot        # one assess call: every captured kernel
    def insts(m):
        return num(m.get(("Instruction Statistics", "Executed Instructions"), ("", ""))[0]) or 0.0
    s["kernels"] = [{"name": dk[k][1].split("(")[0], "duration_ms": dur_ms(dk[k][0]),
                     "dram_bytes": (per[i].get("dram__bytes_read.sum") or 0) + (per[i].get("dram__bytes_write.sum") or 0),
                     "executed_instructions": insts(dk[k][0])}
                    for i, k in enumerate(order)]
    s["executed_instructions_per_call"] = sum(kk["executed_instructions"] for kk in s["kernels"])
    if a.launches:
        s["launch_shares"] = launches(a.launches)
    s["hot_lines"] = hot_lines(a.rep)
    txt = json.dumps(s, indent=1)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")


if __name__ == "__main__":
    main()
