cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_offspring_gpu.py tests/test_stiff_parity.py -m gpu -q -x --durations=10 > gpurun_out/pytest_r2c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2c.log
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_stiff_parity.py > gpurun_out/pytest_r2c_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2c_all.log
