"""A/B timing of two builds of libpfsmc_gpu.so on the same GPU box.

    python profiles/ab.py A.so B.so [rounds] [-- bench args]

Alternates `bench.py --no-cpu-baseline --no-workloads` runs between the two
libraries (PFSMC_GPU_LIB) and prints each headline ms/step and per-kernel time,
then the medians. Used for every "measured back to back, alternating builds"
note in r01_notes.md.
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(lib, extra):
    env = dict(os.environ, PFSMC_GPU_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline",
                          "--no-workloads", *extra], env=env, capture_output=True, text=True,
                         check=True).stdout
    line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
    return line["ms_per_step"], line.get("kernel_ms_per_step", {})


def main():
    argv = sys.argv[1:]
    extra = []
    if "--" in argv:
        i = argv.index("--")
        argv, extra = argv[:i], argv[i + 1:]
    libs = argv[:2]
    rounds = int(argv[2]) if len(argv) > 2 else 3
    res = {lib: [] for lib in libs}
    for r in range(rounds):
        for lib in (libs if r % 2 == 0 else libs[::-1]):
            ms, ker = run(lib, extra)
            res[lib].append((ms, ker))
            print(f"{os.path.basename(lib):>24s} step {ms:.4f} ms  " +
                  "  ".join(f"{k} {v * 1e3:.1f}" for k, v in ker.items()), flush=True)
    for lib in libs:
        ms = statistics.median(m for m, _ in res[lib])
        keys = res[lib][0][1].keys()
        ker = {k: statistics.median(x[1][k] for x in res[lib]) for k in keys}
        print(f"median {os.path.basename(lib):>17s} step {ms:.4f} ms  " +
              "  ".join(f"{k} {v * 1e3:.1f}" for k, v in ker.items()))


if __name__ == "__main__":
    main()
