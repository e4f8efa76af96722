cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python profiles/ab_chain.py ab/base.so ab/rob.so 2 4194304 robertson exact > gpurun_out/ab_rob1.txt 2>&1
timeout 900 python profiles/ab_chain.py ab/base.so ab/rob2.so 2 4194304 robertson exact > gpurun_out/ab_rob2.txt 2>&1
