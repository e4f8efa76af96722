cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r5x.txt 2>&1
timeout 1700 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_r5x.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r5x.log
tail -3 gpurun_out/pytest_r5x.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r5x.log 2>&1
echo "smoke rc=$?" | tee -a gpurun_out/smoke_r5x.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r5x.json 2> gpurun_out/bench_r5x.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r5x_ref.json 2> gpurun_out/bench_r5x_ref.err
echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r5x.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict|k_scan|k_serve" -s 20 -c 8 -o /tmp/r5x_lv python profiles/probe_scanmode.py lv > /dev/null 2>&1
ncu -i /tmp/r5x_lv.ncu-rep --page raw --csv > gpurun_out/r5x_lv_raw.csv 2>&1
python profiles/ncu_lines.py /tmp/r5x_lv.ncu-rep k_scan_fused 40 > gpurun_out/r5x_lines_k_scan_fused.txt 2>&1
du -sh gpurun_out
