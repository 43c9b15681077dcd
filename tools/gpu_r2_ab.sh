# A/B of tuning builds on the configs[3] headline (bench.py, no secondary keys)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARIANTS:-A B C D}; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-secondary} --no-e2e --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json,sys
try:
    l=json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
    print(sys.argv[1], "step", l["ms_per_step"], "GBs", l["value"], "kspec", l["roofline"]["kernel_ms"], "clk", l["clocks"]["sm_mhz"], "halo", l["path"]["halo_chunks"], "fetched", l["roofline"].get("algorithmic_gb_per_launch"), "frac", l["roofline"]["frac"])
    if "configs1" in l: print("   c1", l["configs1"]["ms_per_step"], l["configs1"]["roofline"]["kernel_ms"], "| c4", l["configs4_sharded"]["ram"]["ms_per_step"], l["configs4_sharded"]["ae_max"]["ms_per_step"])
except Exception as e:
    print(sys.argv[1], "FAILED", e); print(open(f"gpurun_out/ab_{sys.argv[1]}.log").read()[-2000:])
PY
done
