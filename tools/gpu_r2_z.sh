# round-2 re-entry check: smoke, the whole -m gpu suite, the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/z_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/z_pytest.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/z_pytest.log
timeout 600 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo bench rc=$?

cut -c1-600 gpurun_out/z_bench.json
