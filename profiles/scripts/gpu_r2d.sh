cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
timeout 300 python profiles/probe_scan.py > gpurun_out/probe_scan_r2d.txt 2>&1
# launch list (cold, serialised) of the headline command
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2d.csv python bench.py --steps 3 --warmup 3 --no-workloads --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
# full captures of the stiff propagation kernels (FP64 pipe evidence), exact and fast
for a in exact fast; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 2 -c 1 -o gpurun_out/r02_chain_${a} python profiles/probe_stiff.py chain $a 22 > gpurun_out/ncu_chain_${a}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 200 -c 1 -o gpurun_out/r02_robertson_${a} python profiles/probe_stiff.py robertson $a 22 > gpurun_out/ncu_rob_${a}.log 2>&1
done
# LV headline kernels
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_predict|k_scan|k_serve" -s 20 -c 5 -o gpurun_out/r02_lv_exact python profiles/probe_scan.py > gpurun_out/ncu_lv.log 2>&1
ls -la gpurun_out
