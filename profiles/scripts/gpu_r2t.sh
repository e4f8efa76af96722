cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2t.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-workloads --no-cpu-baseline > gpurun_out/bench_r2t.json 2> gpurun_out/bench_r2t.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2t.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
