cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python profiles/ab_lv.py ab/base.so ab/storeg.so 3 > gpurun_out/ab_storeg.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lockstep or free_running or fixture or resample" > gpurun_out/pytest_r2y.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2y.log
