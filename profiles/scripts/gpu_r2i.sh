cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 2 -c 1 -o /tmp/r02_chain_fast_src python profiles/probe_stiff.py chain fast 20 > /dev/null 2>&1
ncu -i /tmp/r02_chain_fast_src.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_chain_fast_source.csv 2>&1
ncu -i /tmp/r02_chain_fast_src.ncu-rep --page source --csv > gpurun_out/r02_chain_fast_sass.csv 2>&1
ls -la gpurun_out
