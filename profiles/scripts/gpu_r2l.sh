cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in exact fast; do
timeout 600 python profiles/ab_chain.py ab/new.so ab/new3.so 2 4194304 chain $a > gpurun_out/ab2_chain_$a.txt 2>&1
done
timeout 600 python profiles/ab_chain.py ab/old.so ab/new3.so 2 1048576 lv exact > gpurun_out/ab2_lv_exact.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/old.so ab/new3.so 2 1048576 metabolic exact > gpurun_out/ab2_met_exact.txt 2>&1
timeout 900 python -m pytest tests/test_stiff_parity.py tests/test_gpu_parity.py -m gpu -q -x -k "chain or lockstep or stiff or fixture or metabolic" > gpurun_out/pytest_r2l.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2l.log
