"""Summarise an ncu report (development tool): key raw metrics + top source lines.

usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex] > profiles/<name>.md
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct", "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    print(f"# ncu summary: `{rep}`\n")
    for row in raw[2:]:
        name = row[hdr.index("Kernel Name")]
        if len(sys.argv) > 2 and not re.search(sys.argv[2], name):
            continue
        print(f"## {name}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {m} | {row[i]} | {units[i]} |")
        print()
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    hdr_i = next((i for i, r in enumerate(src) if r and r[0] == "Line No"), None)
    if hdr_i is None:
        return
    h = src[hdr_i]
    iS, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    lines = []
    for r in src[hdr_i + 1:]:
        if len(r) > iI and r[2] == "-" and r[0].isdigit():
            try:
                lines.append((int(r[iS]), int(r[iI]), int(r[0]), r[1].strip()[:100]))
            except ValueError:
                pass
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    print("## top source lines (share of stall samples / executed instructions)\n")
    print("| samples % | inst % | line | source |\n|---|---|---|---|")
    for s, i, ln, txt in sorted(lines, reverse=True)[:25]:
        print(f"| {100 * s / ts:.1f} | {100 * i / ti:.1f} | {ln} | `{txt.replace('|', '/')}` |")


if __name__ == "__main__":
    main()
