cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c5" > gpurun_out/pytest_r2h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2h.log
timeout 300 python profiles/probe_c5_search.py both 5 > gpurun_out/probe_c5_r2h.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r2h.csv python profiles/probe_c5_search.py both 2 > /dev/null 2>&1
