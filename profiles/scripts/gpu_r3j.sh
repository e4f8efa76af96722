cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python profiles/probe_literal.py > gpurun_out/probe_literal2.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r3j.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r3j.log
