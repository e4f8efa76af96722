cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python profiles/probe_literal.py > gpurun_out/probe_literal.txt 2>&1
