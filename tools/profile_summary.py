"""Turn one tools/gpu_round.sh run (gpurun_out/) into the committed profile
artifacts for a version tag (diagnostic tooling, not a measurement):

    python tools/profile_summary.py r01_v10

writes profiles/<tag>_bench.jsonl (the bench line), <tag>_launches.csv (the ncu
launch list), <tag>_k_speculate_details.csv (ncu --page details of the full
capture), and refreshes profiles/ncu_k_speculate_latest.json (the DRAM traffic
bench.py reports).  Prints the numbers the summary markdown quotes.
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
tag = sys.argv[1]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kname = vals[hdr.index("Kernel Name")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    d = {}
    for k, u, v in zip(hdr, units, vals):
        try:
            d[k] = float(v.replace(",", "")) * scale.get(u, 1)  # bytes and nanoseconds
        except ValueError:
            pass
    return kname, d


bench = open(os.path.join(OUT, "bench.log")).read().strip().splitlines()[-1]
json.loads(bench)
with open(os.path.join(PROF, f"{tag}_bench.jsonl"), "w") as f:
    f.write(bench + "\n")
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
rep = os.path.join(OUT, "prof_spec.ncu-rep")
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
with open(os.path.join(PROF, f"{tag}_k_speculate_details.csv"), "w") as f:
    f.write(det)
kname, m = raw_metrics(rep)
rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
latest = {
    "kernel": kname.split("(")[0].replace("void ", "").replace("cdc::", "") + " (configs[1] AE-Max)",
    "version": tag,
    "workload": "configs[1] bench.py --steps 3 --warmup 3 --no-cpu-baseline",
    "capture": "ncu --set full --clock-control none --import-source on, one launch after 3 warm-up steps",
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "traffic_bytes": rd + wr,
    "algorithmic_bytes": 268435456,
    "gpu_time_us": m["gpu__time_duration.sum"] / 1e3,
    "warps_active_pct": m.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": m.get("launch__registers_per_thread"),
    "issue_slots_busy_pct": m.get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "executed_instructions": m.get("smsp__inst_executed.sum"),
}
with open(os.path.join(PROF, "ncu_k_speculate_latest.json"), "w") as f:
    json.dump(latest, f, indent=1)
print(json.dumps(latest, indent=1))
# the launch list: per-kernel time and share of one step
times = {}
for r in csv.reader(open(os.path.join(OUT, "launches.csv"))):
    if len(r) > 14 and r[12] == "gpu__time_duration.sum":
        name = r[4].split("(")[0].replace("void ", "").split("<")[0].replace("cdc::", "")
        times.setdefault(name, []).append(float(r[14]) / 1e3)
for k, v in times.items():
    print(f"launches: {k:30s} n={len(v):3d} mean {sum(v) / len(v):8.2f} us")
