# k_maxp_scan block filter: MAXP parity, timing A/B against the previous build, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_maxp.py -x -q --tb=short -p no:cacheprovider > gpurun_out/mx_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/mx_pytest.log
echo new; timeout 300 python tools/maxp_timing.py
echo old; CDC_LIB=$PWD/build/libcdc_old.so timeout 300 python tools/maxp_timing.py
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_maxp -c 12 --csv --log-file gpurun_out/mx7_launches.csv python tools/maxp_timing.py > /dev/null 2>&1; echo ncu rc=$?
