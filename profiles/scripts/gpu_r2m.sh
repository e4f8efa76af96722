cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python profiles/ab_chain.py ab/new.so ab/new4.so 2 4194304 chain fast > gpurun_out/ab3_chain_fast_4.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/new.so ab/new5.so 2 4194304 chain fast > gpurun_out/ab3_chain_fast_5.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/new4.so ab/new5.so 2 4194304 chain exact > gpurun_out/ab3_chain_exact_45.txt 2>&1
