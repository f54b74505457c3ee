"""Summarise ncu --set full captures into profiles/ text files."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Registers Per Thread", "Grid Size", "Block Size",
        "Achieved Occupancy", "Dynamic Shared Memory Per Block", "L2 Hit Rate",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "SM Frequency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(out.splitlines())
    hdr = next(r)
    lines, name = [], None
    for row in r:
        d = dict(zip(hdr, row))
        name = d["Kernel Name"]
        if d["Metric Name"] in KEYS:
            lines.append(f"  {d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(out.splitlines())
    hdr, units, vals = next(r), next(r), next(r)
    for h, u, v in zip(hdr, units, vals):
        if h in RAW:
            lines.append(f"  {h:40s} {v} {u}")
    return name, lines


if __name__ == "__main__":
    dst, header = sys.argv[1], sys.argv[2]
    with open(dst, "w") as f:
        f.write(header.rstrip() + "\n")
        for rep in sys.argv[3:]:
            name, lines = summary(rep)
            f.write(f"# {rep.split('/')[-1]}\nkernel: {name}\n" + "\n".join(lines) + "\n")
