"""Refresh profiles/r02_phaseB.json['3'] from an `ncu --set full` report of k_phaseB (config 3,
STMF_BATCH=256) and the launch list of one sweep-2 window:
    python tools/update_phaseB_json.py phaseB.ncu-rep launches.csv "capture description"
The previous entry is kept under the key given as 4th argument (default '3_before')."""
import csv
import json
import subprocess
import sys

rep, lst, desc = sys.argv[1], sys.argv[2], sys.argv[3]
keep = sys.argv[4] if len(sys.argv) > 4 else "3_before"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
d = dict(zip(rr[0], rr[2]))
f = lambda k: float(d[k].replace(",", ""))
dur_unit = dict(zip(rr[0], rr[1]))["gpu__time_duration.sum"]
dur = f("gpu__time_duration.sum") * {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6}.get(dur_unit, 1e3)
lines = [l for l in open(lst) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[1:]:
    if len(r) >= len(h) and "k_phaseB" in r[ik]:
        per.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", "")) if r[iv] else 0.0
nb = len(per)
dram = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values()) / nb
tavg = sum(v.get("gpu__time_duration.sum", 0) for v in per.values()) / nb / 1e3
path = "profiles/r02_phaseB.json"
J = json.load(open(path))
J[keep] = J["3"]
J["3"] = {"kernel": "k_phaseB<float,2>", "warp_instructions": f("smsp__inst_executed.sum"), "evals": 512,
          "given": J[keep]["given"], "duration_us": dur,
          "l1_wavefront_frac": f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed") / 100,
          "issue_slots_busy": f("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
          "l1_global_ld_sectors": f("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
          "l1_global_ld_wavefronts": f("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum"),
          "l1_local_ld_wavefronts": f("l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum"),
          "dram_bytes": dram, "dram_bytes_launches": nb, "launch_avg_us_under_ncu": tavg, "capture": desc}
json.dump(J, open(path, "w"), indent=1)
print(json.dumps(J["3"], indent=1))
