"""Instruction mix of one kernel from an ncu SASS source page export
(`ncu -i rep --page source --csv`): executed warp instructions per opcode
family, stall samples per family.

  python profiles/sass_mix.py <source.csv> [top]
"""
import collections
import csv
import sys


def family(op):
    op = op.split(".")[0]
    if op.startswith("D") and op in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
        return op
    return op


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    inst = collections.Counter()
    stall = collections.Counter()
    for r in rows:
        if len(r) <= ei or not r[0].startswith("0x"):
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        try:
            inst[family(op)] += float(r[ei] or 0)
            stall[family(op)] += float(r[st] or 0)
        except ValueError:
            pass
    tot, tots = sum(inst.values()), max(sum(stall.values()), 1)
    fp64 = sum(v for k, v in inst.items() if k in ("DFMA", "DMUL", "DADD"))
    print(f"total warp instructions {tot:.4g}; FP64 arithmetic (DFMA/DMUL/DADD) {100 * fp64 / tot:.1f}%")
    for k, v in inst.most_common(top):
        print(f"{k:12s} {100 * v / tot:6.2f}% inst {100 * stall[k] / tots:6.2f}% stall")


if __name__ == "__main__":
    main()
