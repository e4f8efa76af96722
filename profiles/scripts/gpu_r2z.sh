cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python profiles/ab_lv.py ab/base.so ab/noepi.so 2 > gpurun_out/ab_noepi.txt 2>&1
