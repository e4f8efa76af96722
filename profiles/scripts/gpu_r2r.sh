cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sharded_c5_gpu.py tests/test_gpu_parity.py tests/test_offspring_gpu.py tests/test_sharded.py -m gpu -q -x -k "c5 or shard or offspring" > gpurun_out/pytest_r2r.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2r.log
timeout 600 python bench.py --force-sharded --config 5 --steps 5 --warmup 3 > gpurun_out/bench_c5_sharded_w1.json 2> gpurun_out/bench_c5_sharded_w1.err
timeout 600 python bench.py --force-sharded --config 2 --steps 20 --warmup 5 > gpurun_out/bench_lv_sharded_w1.json 2> gpurun_out/bench_lv_sharded_w1.err
