"""Key metrics of an ncu --set full report (one line per profiled launch)."""
import csv, subprocess, sys

KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "L1/TEX Cache Throughput",
        "L2 Cache Throughput"]

def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    by = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            by.setdefault((d["ID"], d["Kernel Name"][:40]), {})[d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
    for (i, k), m in by.items():
        print(f"launch {i} {k}")
        for key in KEYS:
            if key in m:
                print(f"   {key}: {m[key]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if rr:
        h = rr[0]
        for r in rr[2:]:
            d = dict(zip(h, r))
            rd = d.get("dram__bytes_read.sum"); wr = d.get("dram__bytes_write.sum")
            print(f"   dram read {rd} write {wr} (units row: {dict(zip(h, rr[1])).get('dram__bytes_read.sum')})")

if __name__ == "__main__":
    main(sys.argv[1])
