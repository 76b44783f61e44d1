"""Summarise an ncu report (run here, no GPU needed) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
    "L2 Hit Rate", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Issued Warp Per Scheduler",
    "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
    "Avg. Active Threads Per Warp", "Executed Instructions", "Registers Per Thread", "Block Size", "Grid Size",
    "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy", "Branch Efficiency",
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "gpu__time_duration.sum", "launch__registers_per_thread"]


def main(rep, out):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    lines = [f"# ncu summary of {rep}"]
    kname = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", kname)
        if d.get("Metric Name") in KEYS:
            lines.append(f"{d['Section Name']:32s} {d['Metric Name']:38s} {d['Metric Value']:>16s} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        h, units = rr[0], rr[1]
        for r in rr[2:]:
            for k in RAW:
                if k in h:
                    i = h.index(k)
                    lines.append(f"raw {k:50s} {r[i]:>16s} {units[i]}")
    lines.insert(1, f"# kernel: {kname}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
