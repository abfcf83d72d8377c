"""Summarise an ncu --set full report into a small text file for profiles/:
key throughput/occupancy/memory metrics, warp-stall breakdown and the hottest
SASS instructions (stall samples).  usage: ncu_summary.py REPORT.ncu-rep OUT.txt [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout


def main(rep, out, kernel=None):
    filt = ["-k", "regex:" + kernel] if kernel else []
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"] + filt))))
    h, u, v = raw[0], raw[1], raw[2]
    lines = ["# ncu --set full summary of %s" % rep.split("/")[-1], "# kernel: %s" % v[h.index("Kernel Name")], ""]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append("%-70s %s %s" % (k, v[i], u[i]))
    lines += ["", "# warp stalls (warps per issue-active cycle)"]
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    for val, n in sorted(st, reverse=True)[:10]:
        lines.append("  %-28s %.2f" % (n, val))
    src = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + filt))))
    hi = next(i for i, r in enumerate(src) if r and r[0] == "Address")  # the first kernel's table
    hh = src[hi]
    iE, iS = hh.index("Instructions Executed"), hh.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in src[hi + 1:]:
        if not r or r[0] == "Kernel Name":
            break
        data.append(r)
    tot = sum(int(r[iS]) for r in data) or 1
    totE = sum(int(r[iE]) for r in data)
    lines += ["", "# hottest SASS (stall samples, share, executions); total samples %d, executed %d" % (tot, totE)]
    base = int(data[0][0], 16)
    for r in sorted(data, key=lambda r: -int(r[iS]))[:25]:
        lines.append("  %05x %6d %5.1f%% %10s  %s" % (int(r[0], 16) - base, int(r[iS]), 100.0 * int(r[iS]) / tot, r[iE], r[1].strip()))
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
