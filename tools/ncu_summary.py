"""One-screen summary of an ncu --set full report (details + a few raw counters)."""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Grid Size", "Block Size")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
       "sm__sass_thread_inst_executed_op_dadd_pred_on.sum")


def run(rep):
    out = []
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    isec, iname, iunit, ival = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    kname = h.index("Kernel Name")
    out.append(f"kernel: {rows[1][kname][:110]}")
    seen = set()
    for r in rows[1:]:
        if r[iname] in KEYS and r[iname] not in seen:
            seen.add(r[iname])
            out.append(f"  {r[iname]:36s} {r[ival]:>14s} {r[iunit]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    for k in RAW:
        if k in rr[0]:
            i = rr[0].index(k)
            out.append(f"  {k:60s} {rr[2][i]:>14s} {rr[1][i]}")
    return "\n".join(out)


if __name__ == "__main__":
    title = sys.argv[2] if len(sys.argv) > 2 else ""
    print(("# " + title + "\n" if title else "") + run(sys.argv[1]))
