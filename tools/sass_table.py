#!/usr/bin/env python
"""Per-kernel SASS opcode / register / spill table of the built library
(profiles/r2_sass_table.md): static instruction counts from `cuobjdump -sass`
(DMMA = FP64 tensor core, DFMA/DMUL/DADD = FP64 pipe, UBLKCP = cp.async.bulk
(TMA-class bulk copy), SHFL, BAR) and registers / spill bytes / shared memory
from the ptxas log of the build (build/ptxas.log).

usage: python tools/sass_table.py [out.md]
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2307_16894_b200" / "libpodecm_cuda.so"
OPS = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "UBLKCP", "LDGSTS", "SHFL", "BAR", "LDL", "STL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    counts = defaultdict(Counter)
    fn = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if fn and m:
            counts[fn][m.group(1)] += 1
    regs = {}
    log = (ROOT / "build" / "ptxas.log").read_text() if (ROOT / "build" / "ptxas.log").exists() else ""
    cur = None
    for line in log.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if cur and m and "spill" not in regs.get(cur, {}):  # the entry's own (callees follow)
            regs.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers", line)
        if cur and m:
            sm = re.search(r"(\d+) bytes smem", line)
            regs.setdefault(cur, {}).update(regs=int(m.group(1)), smem=int(sm.group(1)) if sm else 0)
    names = demangle(sorted(counts))
    rows = []
    for f in sorted(counts, key=lambda k: names[k]):
        c = counts[f]
        nm = names[f].replace("(anonymous namespace)::", "")
        nm = re.sub(r"\(.*", "", nm) if "<" not in nm else nm.split("(")[0]
        r = regs.get(f, {})
        rows.append((nm, r.get("regs", ""), r.get("spill", ""), r.get("smem", ""), sum(c.values()),
                     *[c.get(o, 0) for o in OPS]))
    hdr = ["kernel", "regs", "spill st/ld B", "smem B", "SASS"] + OPS
    lines = ["# SASS opcode table (static counts), registers and spills — round 2", "",
             f"Library: `paper_2307_16894_b200/libpodecm_cuda.so` (sm_100a), `cuobjdump -sass` + `build/ptxas.log`.",
             "DMMA is the FP64 tensor-core instruction (`mma.sync.m8n8k4.f64`; tcgen05 has no f64 kind), "
             "UBLKCP the cp.async.bulk copy.", "",
             "| " + " | ".join(hdr) + " |", "|" + "---|" * len(hdr)]
    for r in rows:
        lines.append("| " + " | ".join(str(x) for x in r) + " |")
    out = "\n".join(lines) + "\n"
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(out)
    print(out)


if __name__ == "__main__":
    main()
