cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python profiles/ab_lv.py ab/base.so ab/pdl.so 3 > gpurun_out/ab_pdl.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r3e.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r3e.log
