"""Key metrics of an ncu --set full report (one block per profiled launch)."""
import csv, subprocess, sys

KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "L1/TEX Cache Throughput",
        "L2 Cache Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    by = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            by.setdefault((d["ID"], d["Kernel Name"][:60]), {})[d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rh, ru = rr[0], rr[1]
    for n, ((i, k), m) in enumerate(by.items()):
        print(f"launch {i} {k}")
        for key in KEYS:
            if key in m:
                print(f"   {key}: {m[key]}")
        if 2 + n < len(rr):
            d = dict(zip(rh, rr[2 + n]))
            u = dict(zip(rh, ru))
            for key in RAW:
                if key in d:
                    print(f"   {key}: {d[key]} {u.get(key, '')}")


if __name__ == "__main__":
    main(sys.argv[1])
