cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python profiles/ab_lv.py ab/base.so ab/acqrel.so 3 > gpurun_out/ab_acqrel.txt 2>&1
timeout 900 python profiles/ab_lv.py ab/base.so ab/notree.so 2 > gpurun_out/ab_notree.txt 2>&1
