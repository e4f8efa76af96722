"""Summarise an ncu --csv launch list (time + DRAM bytes per kernel)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rec = dict(zip(hdr, r))
            d[rec["Kernel Name"][:50]][rec["Metric Name"]].append(float(rec["Metric Value"].replace(",", "")))
    for k, v in d.items():
        t = v["gpu__time_duration.sum"]
        rd = v.get("dram__bytes_read.sum", [0])
        wr = v.get("dram__bytes_write.sum", [0])
        n = len(t)
        T = sum(t) / n
        print(f"{k:50s} n={n} {T / 1e3:9.1f}us rd={sum(rd) / n / 1e6:8.1f}MB wr={sum(wr) / n / 1e6:8.1f}MB "
              f"{(sum(rd) + sum(wr)) / n / T:6.0f}GB/s")


if __name__ == "__main__":
    main(sys.argv[1])
