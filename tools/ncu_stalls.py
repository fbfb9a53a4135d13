#!/usr/bin/env python
"""Warp-stall breakdown of an ncu report from its SASS source page (no GPU needed).

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [--kernel N] [--top 25]

Prints, per captured kernel: the sampled stall reasons summed over all instructions (share of samples), the
instruction mix by opcode (executed warp instructions), and the hottest SASS instructions with their top
stall reasons.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess


def pages(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    blocks, cur = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = [line]
            blocks.append(cur)
        elif cur is not None:
            cur.append(line)
    res = []
    for b in blocks:
        name = next(csv.reader([b[0]]))[1]
        rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
        res.append((name, rows[0], rows[1:]))
    return res


def num(v):
    try:
        return float(v)
    except Exception:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", type=int, default=-1)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    for ki, (name, h, rows) in enumerate(pages(a.rep)):
        if a.kernel >= 0 and ki != a.kernel:
            continue
        stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        tot = collections.Counter()
        ops = collections.Counter()
        hot = []
        ci = {c: h.index(c) for c in h}
        for r in rows:
            if len(r) < len(h):
                continue
            for c in stall_cols:
                tot[c] += num(r[ci[c]])
            src = r[ci["Source"]].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1] if len(src.split()) > 1 else op
            ops[op.split(".")[0]] += num(r[ci["Instructions Executed"]])
            hot.append((num(r[ci["# Samples"]]), src, {c: num(r[ci[c]]) for c in stall_cols}))
        S = sum(tot.values()) or 1
        print("== kernel %d: %s" % (ki, name[:90]))
        print("samples %d; stalls:" % S, ", ".join("%s %.1f%%" % (c[6:], 100 * v / S) for c, v in tot.most_common(10)))
        E = sum(ops.values()) or 1
        print("executed warp instructions %.3e; mix:" % E, ", ".join("%s %.1f%%" % (o, 100 * v / E) for o, v in ops.most_common(16)))
        hot.sort(key=lambda t: -t[0])
        for s, src, st in hot[:a.top]:
            top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
            print("  %5.2f%%  %-60s %s" % (100 * s / S, src[:60], " ".join("%s:%d" % (k[6:], v) for k, v in top if v)))


if __name__ == "__main__":
    main()
