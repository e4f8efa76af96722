cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python profiles/ab_chain.py ab/new6.so ab/lv_b256.so 3 1048576 lv exact > gpurun_out/ab5_lv_256.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/lv_b256.so ab/lv_b128.so 3 1048576 lv exact > gpurun_out/ab5_lv_128.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/lv_b256.so ab/lv_b128.so 3 1048576 lv fast > gpurun_out/ab5_lv_128f.txt 2>&1
