cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict" -s 10 -c 2 -o /tmp/r5m_lv python profiles/probe_scanmode.py lv > /dev/null 2>&1
python profiles/ncu_lines.py /tmp/r5m_lv.ncu-rep k_predict 45 > gpurun_out/r5m_lines_k_predict.txt 2>&1
python profiles/ncu_lines.py /tmp/r5m_lv.ncu-rep k_update 60 > gpurun_out/r5m_lines_k_update.txt 2>&1
head -50 gpurun_out/r5m_lines_k_predict.txt
