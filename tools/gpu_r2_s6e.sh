cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/dense_timing.py
N=$((64<<20)) timeout 300 python tools/dense_timing.py
ALGO=ae_max AVG=16384 timeout 300 python tools/dense_timing.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/dn_launches.csv python tools/dense_timing.py > /dev/null 2>&1
python - <<'P'
import csv
for r in list(csv.reader(open('gpurun_out/dn_launches.csv')))[-14:]:
    if len(r) > 14: print(r[4][:60], r[14])
P
