"""Summarise an .ncu-rep: per kernel, the key SOL / memory / scheduler metrics."""
import csv
import io
import subprocess
import sys

KEEP = {
    "GPU Speed Of Light Throughput": ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
                                      "L2 Cache Throughput", "L1/TEX Cache Throughput"],
    "Memory Workload Analysis": ["Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Mem Busy"],
    "Launch Statistics": ["Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
                          "Waves Per SM"],
    "Occupancy": ["Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM"],
    "Scheduler Statistics": ["Issued Warp Per Scheduler", "No Eligible", "Active Warps Per Scheduler",
                             "Eligible Warps Per Scheduler"],
    "Warp State Statistics": ["Warp Cycles Per Issued Instruction"],
    "Compute Workload Analysis": ["Issue Slots Busy", "Executed Ipc Active"],
}


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    idx = {k: h.index(k) for k in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value")}
    cur = None
    lines = []
    for r in rows[1:]:
        kid = (r[idx["ID"]], r[idx["Kernel Name"]][:80])
        if kid != cur:
            cur = kid
            lines.append(f"== kernel {kid[0]}: {kid[1]}")
        sec, name = r[idx["Section Name"]], r[idx["Metric Name"]]
        if sec in KEEP and name in KEEP[sec]:
            lines.append(f"   {sec[:26]:26s} {name:38s} {r[idx['Metric Value']]:>12s} {r[idx['Metric Unit']]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        hh = rr[0]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "gpu__time_duration.sum"]
        cols = [i for i, c in enumerate(hh) if c in want]
        for r in rr[2:]:
            lines.append("   raw: " + ", ".join(f"{hh[i]}={r[i]}" for i in cols))
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
