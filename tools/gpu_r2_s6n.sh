cd $GRAFT_REPO_ROOT
N=$((16<<20)) AVG=8192 K=8 timeout 300 python tools/kphase_timing.py 2>&1 | tail -12
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 12 --csv --log-file gpurun_out/kp_launches.csv env N=$((16<<20)) AVG=8192 K=8 python tools/kphase_timing.py > /dev/null 2>&1
python - <<'P'
import csv
for r in list(csv.reader(open('gpurun_out/kp_launches.csv'))):
    if len(r) > 14 and r[12]=='gpu__time_duration.sum': print(r[4][:50], r[14])
P
