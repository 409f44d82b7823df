"""Summarise an ncu --set full report: key metrics + top stall reasons + top SASS lines.

    python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.max"]
STALLS = ["stall_barrier", "stall_branch_resolving", "stall_long_sb", "stall_math", "stall_mio", "stall_no_inst",
          "stall_not_selected", "stall_selected", "stall_short_sb", "stall_wait", "stall_lg", "stall_membar",
          "stall_dispatch", "stall_sleep"]


def ncu(path, *args):
    return subprocess.run(["ncu", "-i", path, *args], capture_output=True, text=True).stdout


def main(path):
    rows = list(csv.reader(io.StringIO(ncu(path, "--page", "raw", "--csv"))))
    h, u = rows[0], rows[1]
    print("# ncu --set full summary of %s" % path.split("/")[-1])
    for n, v in enumerate(rows[2:]):  # one block per captured launch
        print("\n## launch %d" % n)
        for k in KEYS:
            if k in h:
                print("%-62s %s %s" % (k, v[h.index(k)], u[h.index(k)]))
    # source page: the first captured launch
    src = list(csv.reader(io.StringIO(ncu(path, "--page", "source", "--csv", "--print-source", "sass"))))
    sh, sd = src[1], src[2:]
    idx = {n: sh.index(n) for n in STALLS if n in sh}
    agg = collections.Counter()
    for r in sd:
        for n, i in idx.items():
            if i < len(r) and r[i].isdigit():
                agg[n] += int(r[i])
    tot = sum(agg.values()) or 1
    print("\nwarp stall samples (share):")
    for n, c in agg.most_common():
        if c:
            print("  %-24s %6d  %5.1f%%" % (n, c, 100.0 * c / tot))
    iS, iE, iW = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
    print("\ntop SASS lines by stall samples (executed, samples, instruction):")
    sd = [r for r in sd if len(r) > max(iS, iE, iW)]
    for r in sorted(sd, key=lambda r: -int(r[iW]) if r[iW].isdigit() else 0)[:15]:
        print("  %10s %6s  %s" % (r[iE], r[iW], r[iS].strip()[:90]))


if __name__ == "__main__":
    main(sys.argv[1])
