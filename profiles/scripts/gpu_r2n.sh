cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python profiles/ab_chain.py ab/new.so ab/new6.so 2 4194304 chain fast > gpurun_out/ab4_chain_fast.txt 2>&1
timeout 600 python profiles/ab_chain.py ab/new.so ab/new6.so 2 4194304 chain exact > gpurun_out/ab4_chain_exact.txt 2>&1
