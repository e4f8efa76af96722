"""Key per-kernel metrics from an ncu report: duration, DRAM bytes,
achieved occupancy, issue activity, instruction count, FP64 pipe.

  python profiles/ncu_summary.py <report.ncu-rep | raw page .csv>
(a .csv is the output of `ncu -i report --page raw --csv`, exported on the
GPU box so the large report need not travel)
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "dur_us", 1e-3),
        ("dram__bytes_read.sum", "dram_rd_MB", 1e-6),
        ("dram__bytes_write.sum", "dram_wr_MB", 1e-6),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occup_%", 1),
        ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue_%", 1),
        ("smsp__inst_executed.sum", "warp_inst_M", 1e-6),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_%", 1),
        ("launch__registers_per_thread", "regs", 1),
        ("launch__grid_size", "grid", 1),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%", 1)]


def main():
    if sys.argv[1].endswith(".csv"):
        out = open(sys.argv[1]).read()
    else:
        out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    while rows and "Kernel Name" not in rows[0]:
        rows = rows[1:]
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    print(f"{'kernel':44s} " + " ".join(f"{k[1]:>11s}" for k in KEYS))
    for r in rows[2:]:
        vals = []
        for name, short, scale in KEYS:
            if name in hdr:
                v = r[hdr.index(name)].replace(",", "")
                u = units[hdr.index(name)]
                try:
                    x = float(v)
                    if name.startswith("dram__bytes"):
                        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
                    if name == "gpu__time_duration.sum":  # -> ns, then dur_us = ns * 1e-3
                        x *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}.get(u, 1)
                    vals.append(f"{x * scale:11.2f}")
                except ValueError:
                    vals.append(f"{v:>11s}")
            else:
                vals.append(f"{'-':>11s}")
        print(f"{r[ki][:44]:44s} " + " ".join(vals))


if __name__ == "__main__":
    main()
