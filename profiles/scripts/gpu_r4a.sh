cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_r4a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r4a.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke_r4a.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r4a.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r4a.json 2> gpurun_out/bench_r4a.err
echo "bench rc=$?"
