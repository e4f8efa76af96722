cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_fused -s 9 -c 1 -o /tmp/r5r_c5 python profiles/probe_fused.py --c5 > /dev/null 2>&1
python profiles/ncu_lines.py /tmp/r5r_c5.ncu-rep k_scan_fused 45 > gpurun_out/r5r_lines_scan_c5.txt 2>&1
ncu -i /tmp/r5r_c5.ncu-rep --page raw --csv > gpurun_out/r5r_c5_raw.csv 2>&1
python profiles/ncu_summary.py gpurun_out/r5r_c5_raw.csv
head -48 gpurun_out/r5r_lines_scan_c5.txt
