#!/usr/bin/env python
"""SASS summary of the built library: per kernel, registers / stack / local bytes (cuobjdump -res-usage) and
the static counts of the instructions that show how it uses the hardware (TMA loads, mbarrier waits, packed
FP32, streaming 128-bit stores, spills, MUFU, shared-memory traffic).  No GPU needed.

    python tools/sass_summary.py [paper_2503_02412_b200/libse2map.so] [--out profiles/r02_sass_summary.json]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# mnemonic prefixes counted (static, per kernel); an entry counts an instruction whose opcode starts with it
OPS = ["UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "FFMA2", "FADD2", "FMUL2", "FFMA", "MUFU", "STG.E.EF.128", "STG",
       "LDG", "LDS", "STS", "LDL", "STL", "SHFL", "BAR", "ATOMS", "RED", "DFMA", "DADD", "DMUL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out)) if len(out) == len(names) else {n: n for n in names}


def res_usage(lib):
    txt = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    res, cur = {}, None
    for line in txt.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        if cur and "REG:" in line:
            res[cur] = {k.lower(): int(v) for k, v in re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", line)}
            cur = None
    return res


def sass_counts(lib):
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    counts, total, cur = {}, collections.Counter(), None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            op = m.group(1)
            total[cur] += 1
            for p in OPS:
                if op == p or op.startswith(p + "."):
                    counts[cur][p] += 1
            if op.startswith("STG.E.EF.128"):
                counts[cur]["STG.E.EF.128"] += 0  # (counted by the prefix rule above)
    return counts, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib", nargs="?", default=os.path.join(ROOT, "paper_2503_02412_b200", "libse2map.so"))
    ap.add_argument("--out")
    a = ap.parse_args()
    res = res_usage(a.lib)
    counts, total = sass_counts(a.lib)
    names = sorted(set(res) | set(counts))
    dm = demangle(names)
    rows = {}
    for n in names:
        r = dict(res.get(n, {}))
        r["instructions"] = total.get(n, 0)
        r["ops"] = dict(sorted(counts.get(n, {}).items()))
        rows[dm[n]] = r
    doc = {"lib": os.path.relpath(a.lib, ROOT), "counted": OPS,
           "note": "static SASS counts per kernel (cuobjdump -sass of the sm_100a cubin); an opcode counts under every "
                   "listed prefix it starts with (STG.E.EF.128 is also an STG); stack / local = bytes per thread",
           "kernels": rows}
    js = json.dumps(doc, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(js + "\n")
    for k, r in rows.items():
        if "assess_kernel" in k or "sdf" in k:
            print(f"{k[:60]:60s} reg {r.get('reg')} stack {r.get('stack')} instr {r['instructions']} {r['ops']}")


if __name__ == "__main__":
    main()
