cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "resample or scan_modes or c5 or free_running" --durations=10 > gpurun_out/pytest_r5a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r5a.log
tail -5 gpurun_out/pytest_r5a.log
timeout 600 python profiles/probe_scanmode.py lv c5 > gpurun_out/scanmode_r5a.json 2> gpurun_out/scanmode_r5a.err
echo "probe rc=$?"
cat gpurun_out/scanmode_r5a.json
tail -5 gpurun_out/scanmode_r5a.err
