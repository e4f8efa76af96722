cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python profiles/probe_cert.py 20 > gpurun_out/probe_cert.txt 2>&1
timeout 300 python profiles/probe_cert.py 16 >> gpurun_out/probe_cert.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "certified or lockstep" > gpurun_out/pytest_r2u.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2u.log
