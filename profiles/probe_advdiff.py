"""The advdiff workload line of bench.py on its own (GPU box):
python profiles/probe_advdiff.py [--no-cpu]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

if __name__ == "__main__":
    fp64 = bench.fp64_peak(0)
    print(json.dumps(bench.bench_advdiff(0, fp64, cpu="--no-cpu" not in sys.argv)))
