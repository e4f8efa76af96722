cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_offspring_gpu.py tests/test_gpu_parity.py tests/test_sharded.py tests/test_sharded_c5_gpu.py -m gpu -q -x -k "offspring or shard" > gpurun_out/pytest_r3k.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r3k.log
timeout 600 python bench.py --force-sharded --config 2 --steps 20 --warmup 5 > gpurun_out/bench_lv_sharded_w1b.json 2> gpurun_out/bench_lv_sharded_w1b.err
