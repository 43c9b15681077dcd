"""Commit the artefacts of one tools/gpu_prof_r2.sh run (gpurun_out/) for a tag
(diagnostic tooling, not a measurement):

    python tools/profile_r2.py r02_c3 prof_c3 ncu_k_speculate_c3.json "configs[3] ..." ALG_BYTES

writes profiles/<tag>_bench.jsonl (the bench line), <tag>_launches.csv (the
ncu launch list of the bench command), <tag>_k_speculate_details.csv (ncu
--page details of the full capture) and profiles/<json> (the DRAM traffic
bench.py reports), and prints the per-kernel launch-list summary.
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag, rep_name, json_name, workload, alg = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5])
rep = os.path.join(OUT, rep_name + ".ncu-rep")


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    d = {}
    for k, u, v in zip(hdr, units, vals):
        try:
            d[k] = float(v.replace(",", "")) * scale.get(u, 1)  # bytes and nanoseconds
        except ValueError:
            pass
    return vals[hdr.index("Kernel Name")], d


bench = open(os.path.join(OUT, "bench.log")).read().strip().splitlines()[-1]
json.loads(bench)
with open(os.path.join(PROF, f"{tag}_bench.jsonl"), "w") as f:
    f.write(bench + "\n")
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
with open(os.path.join(PROF, f"{tag}_k_speculate_details.csv"), "w") as f:
    f.write(det)
kname, m = raw_metrics(rep)
rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
summary = {
    "kernel": kname.split("(")[0].replace("void ", "").replace("cdc::", ""),
    "version": tag,
    "workload": workload,
    "capture": "ncu --set full --clock-control none --import-source on -k regex:k_speculate -s 3 -c 1 "
               "(tools/gpu_prof_r2.sh)",
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "traffic_bytes": rd + wr,
    "algorithmic_bytes": alg,
    "gpu_time_us": m["gpu__time_duration.sum"] / 1e3,
    "warps_active_pct": m.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": m.get("launch__registers_per_thread"),
    "issue_slots_busy_pct": m.get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "executed_instructions": m.get("smsp__inst_executed.sum"),
}
with open(os.path.join(PROF, json_name), "w") as f:
    json.dump(summary, f, indent=1)
print(json.dumps(summary, indent=1))
times = {}
for r in csv.reader(open(os.path.join(OUT, "launches.csv"))):
    if len(r) > 14 and r[12] == "gpu__time_duration.sum":
        name = r[4].split("(")[0].replace("void ", "").split("<")[0].replace("cdc::", "")
        times.setdefault(name, []).append(float(r[14].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in times.values())
for k, v in times.items():
    print(f"launches: {k:30s} n={len(v):3d} mean {sum(v) / len(v):9.2f} us  share {sum(v) / tot:.3f}")
