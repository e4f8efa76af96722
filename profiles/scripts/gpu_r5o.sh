cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r5o_sharded.csv python bench.py --force-sharded --config 2 --steps 4 --warmup 3 > /dev/null 2>&1
python profiles/launch_table.py gpurun_out/launches_r5o_sharded.csv | head -40
