cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python profiles/probe_scan.py --c5 > gpurun_out/probe_scan_r2g.txt 2>&1
