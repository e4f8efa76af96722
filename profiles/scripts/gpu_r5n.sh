cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_r5n.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r5n.log
tail -4 gpurun_out/pytest_r5n.log
timeout 300 python profiles/probe_scanmode.py lv c5 > gpurun_out/scanmode_r5n.json 2>gpurun_out/scanmode_r5n.err
python - <<PY
import json
d=json.load(open("gpurun_out/scanmode_r5n.json"))
for k,v in d.items():
    print(k, v["ms_per_step"] if isinstance(v,dict) else v, v.get("kernel_us") if isinstance(v,dict) else "")
PY
timeout 600 python bench.py --force-sharded --config 2 --steps 20 --warmup 5 > gpurun_out/bench_r5n_sharded_w1.json 2> gpurun_out/bench_r5n_sharded_w1.err
tail -c 1500 gpurun_out/bench_r5n_sharded_w1.json | head -c 600
