"""profiles/kernel_traffic.json from an ncu --set full report: DRAM bytes
(read + write) per launch for each kernel (mean over the captured launches).

  python profiles/make_traffic.py <report.ncu-rep | raw page .csv> [out.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/kernel_traffic.json"
    if rep.endswith(".csv"):  # `ncu -i report --page raw --csv` exported on the GPU box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    while rows and "Kernel Name" not in rows[0]:
        rows = rows[1:]
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    acc = collections.defaultdict(list)
    pct = collections.defaultdict(lambda: collections.defaultdict(list))
    extra = {"issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
             "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
             "warp_inst_per_launch": "smsp__inst_executed.sum"}
    for r in rows[2:]:
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i].replace(",", "")) * UNIT.get(units[i], 1)
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip().split("::")[-1]
        acc[name].append(tot)
        for key, metric in extra.items():
            if metric in hdr:
                pct[name][key].append(float(r[hdr.index(metric)].replace(",", "")))
    res = {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v), "source": rep.split("/")[-1],
               **{key: sum(x) / len(x) for key, x in pct[k].items()}}
           for k, v in acc.items()}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
