# session 6: dense-index mode -- parity and configs[0] timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q --tb=short > gpurun_out/t_dense.log 2>&1; echo dense rc=$?; tail -15 gpurun_out/t_dense.log
timeout 1200 python -m pytest tests/test_gpu_tables.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q --tb=short > gpurun_out/t6d.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/t6d.log
for v in 1 0; do
  echo "== CDC_DENSE=$v"; CDC_DENSE=$v ONLY="c0" timeout 600 python tools/workloads.py 2>&1 | cut -c1-250
done
