# segment-size sweep of bench.py (kernel numbers only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/sweep.log
for seg in ${SEGS:-0 65536 131072 262144}; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --seg-bytes $seg > gpurun_out/b.log 2>&1
  python - "$seg" <<'PY' >> gpurun_out/sweep.log
import json,sys
l=json.loads(open("gpurun_out/b.log").read().strip().splitlines()[-1])
print(sys.argv[1], l["value"], l["roofline"]["achieved"], l["roofline"]["frac"], l["roofline"]["share_of_step"])
PY
done
cat gpurun_out/sweep.log
