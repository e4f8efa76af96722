cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for a in exact fast; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict" -s 2 -c 2 -o /tmp/r02_chain2_${a} python profiles/probe_stiff.py chain $a 22 > /dev/null 2>&1
ncu -i /tmp/r02_chain2_${a}.ncu-rep --page raw --csv > gpurun_out/r02_chain2_${a}_raw.csv 2>&1
ncu -i /tmp/r02_chain2_${a}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_chain2_${a}_source.csv 2>&1
done
