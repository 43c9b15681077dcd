timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_x.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t_x.log
ONLY=c0,u256,c2,c4 timeout 900 python tools/workloads.py 2>&1 | cut -c1-200
echo "== TMODE=0"; CDC_TMODE=0 ONLY=c0,u256 timeout 900 python tools/workloads.py 2>&1 | cut -c1-200
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_x.json 2> gpurun_out/b_x.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/b_x.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step']); print({k: d[k] for k in d if k.startswith('configs')})"
