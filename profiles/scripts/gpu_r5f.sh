cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r5f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r5f.log
tail -16 gpurun_out/pytest_r5f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r5f.log 2>&1
echo "smoke rc=$?"
