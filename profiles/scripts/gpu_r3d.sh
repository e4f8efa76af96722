cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python profiles/ab_chain.py ab/base.so ab/split.so 2 4194304 chain exact > gpurun_out/ab_split_exact.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/base.so ab/split.so 2 4194304 chain fast > gpurun_out/ab_split_fast.txt 2>&1
timeout 900 python -m pytest tests/test_stiff_parity.py tests/test_gpu_parity.py tests/test_sharded.py -m gpu -q -x -k "chain or shard" > gpurun_out/pytest_r3d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r3d.log
