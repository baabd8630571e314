#!/usr/bin/env python
"""Key metrics of an ncu report (one kernel): time, DRAM bytes, throughput, occupancy, issue, stalls."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    print(f"== {rep}: {v[h.index('Kernel Name')][:90]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:60s} {v[i]:>14s} {u[i]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(v[i]), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1
    print("  stall samples: " + ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
