#!/usr/bin/env python
"""Summarise an `ncu --set full` report (raw page) and an ncu launch list into markdown.

    python scripts/ncu_summary.py gpurun_out/prof_sl.ncu-rep [gpurun_out/launches.csv] > profiles/rNN_x.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "kernel time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs), CTAs"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short-scoreboard / issue"),
    ("local_store_bytes", "local (spill) stores"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(r, hdr, units) for r in rows[2:]]


def main():
    rep = sys.argv[1]
    print(f"## ncu --set full: `{rep}`\n")
    for r, hdr, units in raw(rep):
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"### {name}\n\n| metric | value | unit |\n|---|---|---|")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {label} (`{k}`) | {r[i]} | {units[i]} |")
        print()
    if len(sys.argv) > 2:
        print(f"## launch list (`ncu --metrics gpu__time_duration.sum`): `{sys.argv[2]}`\n")
        print("| # | kernel | grid | block | ns |\n|---|---|---|---|---|")
        with open(sys.argv[2]) as f:
            lines = [l for l in f if l.startswith('"')]
        tot, ours = 0, 0
        for row in csv.DictReader(lines):
            v = float(row["Metric Value"])
            name = row["Kernel Name"]
            tot += v
            if "xslp" in name:
                ours += v
            print(f"| {row['ID']} | {name[:70]} | {row['Grid Size']} | {row['Block Size']} | {v:.0f} |")
        print(f"\nxslp kernels: {ours / 1e6:.3f} ms of {tot / 1e6:.3f} ms total "
              f"({100 * ours / max(tot, 1):.1f}%); the remainder is torch (setup, sanity check).")


if __name__ == "__main__":
    main()
