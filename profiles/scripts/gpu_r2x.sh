cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python profiles/ab_tile.py > gpurun_out/ab_tile.txt 2>&1
