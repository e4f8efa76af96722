"""Per-source-line attribution from an ncu report (cuda,sass source view):
instructions executed and warp-stall samples per (file, line).

  python profiles/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr = None, None
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    tot_e = tot_s = 0.0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ei = hdr.index("Instructions Executed")
            si = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr and r[0] and r[0].isdigit():
            try:
                e, s = float(r[ei] or 0), float(r[si] or 0)
            except ValueError:
                continue
            k = (fname, int(r[0]))
            agg[k][0] += e
            agg[k][1] += s
            agg[k][2] = r[1][:70]
            tot_e += e
            tot_s += s
    print(f"total warp-instructions {tot_e:.0f}, stall samples {tot_s:.0f}")
    for k, (e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]:16s}:{k[1]:<5d} {100*e/tot_e:5.1f}% inst {100*s/max(tot_s,1):5.1f}% stall | {src}")


if __name__ == "__main__":
    main()
