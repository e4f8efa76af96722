cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in base t11; do
PFSMC_GPU_LIB=ab/$lib.so timeout 300 python profiles/probe_c5_search.py split 5 > gpurun_out/c5_$lib.txt 2>&1
PFSMC_GPU_LIB=ab/$lib.so timeout 300 python profiles/probe_c5_search.py guide 5 >> gpurun_out/c5_$lib.txt 2>&1
done
timeout 600 python profiles/ab_chain.py ab/base.so ab/t11.so 2 16777216 chain exact > gpurun_out/ab_t11_chain.txt 2>&1
PFSMC_GPU_LIB=ab/t11.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c5" > gpurun_out/pytest_t11.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_t11.log
