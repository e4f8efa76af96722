cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict" -s 2 -c 2 -o /tmp/r02_chain3_fast python profiles/probe_stiff.py chain fast 22 > /dev/null 2>&1
ncu -i /tmp/r02_chain3_fast.ncu-rep --page raw --csv > gpurun_out/r02_chain3_fast_raw.csv 2>&1
ncu -i /tmp/r02_chain3_fast.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_chain3_fast_source.csv 2>&1
