cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_c5_gpu.py tests/test_gpu_parity.py -m gpu -q -x -k "c5 or sharded" > gpurun_out/pytest_r2q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2q.log
timeout 600 python bench.py --force-sharded --config 5 --steps 5 --warmup 3 > gpurun_out/bench_c5_sharded_w1.json 2> gpurun_out/bench_c5_sharded_w1.err
