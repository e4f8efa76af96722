cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r2s.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2s.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2s.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r2s.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2s_ref.json 2> gpurun_out/bench_r2s_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2s.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict|k_scan|k_serve" -s 20 -c 5 -o /tmp/r02_lv2 python profiles/probe_scan.py > /dev/null 2>&1
ncu -i /tmp/r02_lv2.ncu-rep --page raw --csv > gpurun_out/r02_lv2_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_update|k_predict" -s 2 -c 2 -o /tmp/r02_chain4_exact python profiles/probe_stiff.py chain exact 22 > /dev/null 2>&1
ncu -i /tmp/r02_chain4_exact.ncu-rep --page raw --csv > gpurun_out/r02_chain4_exact_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_update|k_predict" -s 200 -c 2 -o /tmp/r02_rob2_exact python profiles/probe_stiff.py robertson exact 22 > /dev/null 2>&1
ncu -i /tmp/r02_rob2_exact.ncu-rep --page raw --csv > gpurun_out/r02_rob2_exact_raw.csv 2>&1
