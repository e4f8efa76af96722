cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_stiff_parity.py tests/test_gpu_parity.py tests/test_sharded.py tests/test_offspring_gpu.py -m gpu -q -x > gpurun_out/pytest_r2j.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2j.log
for a in exact fast; do
timeout 600 python profiles/ab_chain.py ab/old.so ab/new.so 2 4194304 chain $a > gpurun_out/ab_chain_$a.txt 2>&1
done
timeout 600 python profiles/ab_chain.py ab/old.so ab/new.so 2 4194304 robertson fast > gpurun_out/ab_rob_fast.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/old.so ab/new.so 2 1048576 lv exact > gpurun_out/ab_lv_exact.txt 2>&1
