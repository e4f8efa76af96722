cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_stiff_parity.py tests/test_gpu_parity.py -m gpu -q --durations=10 > gpurun_out/pytest_r2b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --arithmetic fast > gpurun_out/bench_r2b_fast.json 2> gpurun_out/bench_r2b_fast.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --arithmetic exact > gpurun_out/bench_r2b_exact.json 2> gpurun_out/bench_r2b_exact.err
