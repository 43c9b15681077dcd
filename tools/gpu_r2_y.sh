timeout 900 python -m pytest tests/test_gpu_kphase.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t_y.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t_y.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b_y.json 2> gpurun_out/b_y.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/b_y.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step']); print(d['configs4_sharded'])"
ONLY=c4full timeout 900 python tools/workloads.py 2>&1 | cut -c1-200
