cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "resample or scan_modes or c5 or free_running" > gpurun_out/pytest_r5j.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r5j.log
tail -5 gpurun_out/pytest_r5j.log
timeout 300 python profiles/probe_tiles.py 2>&1 | head -64
timeout 600 python profiles/probe_scanmode.py lv c5 > gpurun_out/scanmode_r5j.json 2> gpurun_out/scanmode_r5j.err
python - <<PY
import json
d=json.load(open("gpurun_out/scanmode_r5j.json"))
for k,v in d.items():
    print(k, v["ms_per_step"] if isinstance(v,dict) else v, v.get("kernel_us") if isinstance(v,dict) else "")
PY
