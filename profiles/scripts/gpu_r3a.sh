cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python profiles/ab_lv.py ab/base.so ab/warpepi.so 3 > gpurun_out/ab_warpepi.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/base.so ab/warpepi.so 2 4194304 chain exact > gpurun_out/ab_warpepi_chain.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r3a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r3a.log
