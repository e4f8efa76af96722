cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r2f.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_r2f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2f.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r2f.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-workloads --arithmetic fast > gpurun_out/bench_r2f_fast.json 2> gpurun_out/bench_r2f_fast.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2f_ref.json 2> gpurun_out/bench_r2f_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2f.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict|k_scan|k_serve" -s 20 -c 5 -o /tmp/r02_lv python profiles/probe_scan.py > /dev/null 2>&1
ncu -i /tmp/r02_lv.ncu-rep --page raw --csv > gpurun_out/r02_lv_raw.csv 2>&1
ncu -i /tmp/r02_lv.ncu-rep --page source --csv > gpurun_out/r02_lv_source.csv 2>&1
for a in exact fast; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 2 -c 1 -o /tmp/r02_chain_${a} python profiles/probe_stiff.py chain $a 22 > /dev/null 2>&1
ncu -i /tmp/r02_chain_${a}.ncu-rep --page raw --csv > gpurun_out/r02_chain_${a}_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 200 -c 1 -o /tmp/r02_rob_${a} python profiles/probe_stiff.py robertson $a 22 > /dev/null 2>&1
ncu -i /tmp/r02_rob_${a}.ncu-rep --page raw --csv > gpurun_out/r02_rob_${a}_raw.csv 2>&1
done
du -sh gpurun_out
