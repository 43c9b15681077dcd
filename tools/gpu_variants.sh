# compare tuning builds under build/ on configs[1] (kernel numbers only) + parity smoke of each
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-A B C D}; do
  export CDC_LIB=$PWD/build/libcdc_$v.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "small_segments or config1 or batch_edge" 2>&1 | tail -1
  timeout 300 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_$v.log 2>&1
  python - "$v" <<'PY'
import json,sys
l=json.loads(open(f"gpurun_out/b_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], "step", l["ms_per_step"], "GBs", l["value"], "kspec", l["roofline"]["kernel_ms"], "frac", l["roofline"]["frac"], "segs", l["path"]["segments"], "fast", l["path"]["fast_path"])
PY
done
