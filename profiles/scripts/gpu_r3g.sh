cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_r3g.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r3g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3g.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_r3g.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r3g.json 2> gpurun_out/bench_r3g.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r3g_ref.json 2> gpurun_out/bench_r3g_ref.err
PFSMC_BENCH_FORCE_SHARD_FAIL=1 timeout 600 python bench.py --force-sharded --steps 5 --warmup 3 --no-workloads --no-cpu-baseline > gpurun_out/bench_r3g_fallback.json 2> gpurun_out/bench_r3g_fallback.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r3g.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict|k_scan|k_serve" -s 20 -c 5 -o /tmp/r02_lv3 python profiles/probe_scan.py > /dev/null 2>&1
ncu -i /tmp/r02_lv3.ncu-rep --page raw --csv > gpurun_out/r02_lv3_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_update|k_predict" -s 2 -c 2 -o /tmp/r02_chain5_fast python profiles/probe_stiff.py chain fast 22 > /dev/null 2>&1
ncu -i /tmp/r02_chain5_fast.ncu-rep --page raw --csv > gpurun_out/r02_chain5_fast_raw.csv 2>&1
