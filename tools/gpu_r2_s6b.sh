# session 6: sparse walk with two speculative copies ahead (default) vs one (build/libcdc_D1.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_kphase.py tests/test_gpu_tables.py -x -q > gpurun_out/t6.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t6.log
B="python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e --no-cpu-baseline"
for v in A D1 A D1; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"
  timeout 600 $B 2>&1 | python -c "import sys,json; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 ms', l['ms_per_step'], 'kernel', l['roofline']['kernel_ms'], 'fetched', l['roofline']['algorithmic_gb_per_launch'], 'frac', l['roofline']['frac'])"
done
for v in A D1; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"; ONLY="c2 c4" timeout 900 python tools/workloads.py 2>&1 | cut -c1-72
done
unset CDC_LIB
for kg in "4 2368" "4 1184" "8 1184" "8 592"; do
  set -- $kg
  echo "== K=$1 G=$2"; CDC_KPHASE=$1 CDC_KSEGS=$2 ONLY=c2 timeout 900 python tools/workloads.py 2>&1 | grep "base" | grep -v " 4096 " | cut -c1-72
done
