cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err
tail -c 3000 gpurun_out/bench_r2e.err
timeout 300 python profiles/probe_scan.py > gpurun_out/probe_scan_r2e.txt 2>&1
timeout 600 python -m pytest tests/test_plugin.py -q > gpurun_out/pytest_plugin.log 2>&1
for a in exact fast; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 2 -c 1 -o /tmp/r02_chain_${a} python profiles/probe_stiff.py chain $a 22 > /dev/null 2>&1
ncu -i /tmp/r02_chain_${a}.ncu-rep --page raw --csv > gpurun_out/r02_chain_${a}_raw.csv 2>&1
ncu -i /tmp/r02_chain_${a}.ncu-rep --page source --csv > gpurun_out/r02_chain_${a}_source.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 200 -c 1 -o /tmp/r02_rob_${a} python profiles/probe_stiff.py robertson $a 22 > /dev/null 2>&1
ncu -i /tmp/r02_rob_${a}.ncu-rep --page raw --csv > gpurun_out/r02_rob_${a}_raw.csv 2>&1
ncu -i /tmp/r02_rob_${a}.ncu-rep --page source --csv > gpurun_out/r02_rob_${a}_source.csv 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict|k_scan|k_serve" -s 20 -c 5 -o /tmp/r02_lv python profiles/probe_scan.py > /dev/null 2>&1
ncu -i /tmp/r02_lv.ncu-rep --page raw --csv > gpurun_out/r02_lv_raw.csv 2>&1
ncu -i /tmp/r02_lv.ncu-rep --page source --csv > gpurun_out/r02_lv_source.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2e.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
du -sh gpurun_out
