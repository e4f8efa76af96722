cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_offspring_gpu.py tests/test_gpu_parity.py tests/test_sharded.py tests/test_sharded_c5_gpu.py -m gpu -q -x -k "offspring or shard" > gpurun_out/pytest_r5p.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r5p.log
tail -3 gpurun_out/pytest_r5p.log
timeout 600 python bench.py --force-sharded --config 2 --steps 20 --warmup 5 > gpurun_out/bench_r5p_sharded_w1.json 2> gpurun_out/bench_r5p_sharded_w1.err
python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/bench_r5p_sharded_w1.json") if l.startswith("{")][-1])
print("sharded w1 ms/step", d["ms_per_step"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r5p_sharded.csv python bench.py --force-sharded --config 2 --steps 4 --warmup 3 > /dev/null 2>&1
python profiles/launch_table.py gpurun_out/launches_r5p_sharded.csv | grep -i "offspring\|k_off"
