cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
s=$(date +%s); timeout 600 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err; echo bench rc=$? secs=$(( $(date +%s) - s ))
cut -c1-3000 gpurun_out/z_bench.json
tail -3 gpurun_out/z_bench.err
