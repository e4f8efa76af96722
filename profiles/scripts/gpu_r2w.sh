cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_serve" -s 20 -c 3 -o /tmp/r02_scan python profiles/probe_scan.py > /dev/null 2>&1
ncu -i /tmp/r02_scan.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_scan_source.csv 2>&1
ncu -i /tmp/r02_scan.ncu-rep --page raw --csv > gpurun_out/r02_scan_raw.csv 2>&1
