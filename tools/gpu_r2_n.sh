# A/B of the lean sparse walk (in-tree lib) against HEAD's (build/libcdc_old.so)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_n.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t_n.log
B="python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e --no-cpu-baseline"
for v in old new old new; do
  if [ $v = old ]; then export CDC_LIB=$PWD/build/libcdc_old.so; else unset CDC_LIB; fi
  timeout 600 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])"
done
for v in old new; do
  if [ $v = old ]; then export CDC_LIB=$PWD/build/libcdc_old.so; else unset CDC_LIB; fi
  echo "== $v"; ONLY=c2,c4 timeout 900 python tools/workloads.py 2>&1 | cut -c1-100
done
