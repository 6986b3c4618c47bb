#!/usr/bin/env python
"""Summarise ncu --set full reports into the metrics the roofline cites.

usage: python tools/ncu_summary.py report.ncu-rep [...]  (needs `ncu` on PATH)
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "dfma_thr"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "dmul_thr"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "dadd_thr"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__t_bytes.sum", "l1_bytes"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("local_load_bytes", "local"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    return hdr, units, data


def main():
    for rep in sys.argv[1:]:
        hdr, units, data = rows(rep)
        idx = {h: i for i, h in enumerate(hdr)}
        print(f"## {rep}")
        for d in data:
            name = d[idx["Kernel Name"]] if "Kernel Name" in idx else "?"
            short = name.split("(")[0].split("::")[-1][:60]
            vals = []
            for k, lab in KEYS:
                if k in idx:
                    vals.append(f"{lab}={d[idx[k]]}{units[idx[k]] if units[idx[k]] not in ('', 'inst', 'thread') else ''}")
            print(f"- {short}: " + ", ".join(vals))
        print()


if __name__ == "__main__":
    main()
