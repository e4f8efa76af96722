cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python profiles/probe_fused.py --c5 > gpurun_out/fused_ts_r5b.txt 2>&1
cat gpurun_out/fused_ts_r5b.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scan_fused" -s 8 -c 4 -o /tmp/r5b python profiles/probe_fused.py --c5 > /dev/null 2>&1
ncu -i /tmp/r5b.ncu-rep --page raw --csv > gpurun_out/r5b_raw.csv 2>&1
python profiles/ncu_lines.py /tmp/r5b.ncu-rep k_scan_fused 40 > gpurun_out/r5b_lines.txt 2>&1
python profiles/ncu_summary.py gpurun_out/r5b_raw.csv > gpurun_out/r5b_summary.txt 2>&1
cat gpurun_out/r5b_summary.txt
