"""Summarise an ncu source page (--page source --csv --print-source sass):
top instructions per stall reason, with the preceding instructions."""
import csv
import sys


def main(path, reasons=("stall_long_sb", "stall_barrier", "stall_wait", "stall_short_sb"), top=8, ctx=3):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = rows[2:]
    isrc, ia = h.index("Source"), h.index("Address")
    tot = sum(int(r[h.index("Warp Stall Sampling (All Samples)")]) for r in data)
    for rs in reasons:
        j = h.index(rs)
        s = sum(int(r[j]) for r in data)
        print(f"== {rs}: {s} samples ({100 * s / max(tot, 1):.1f}%)")
        idx = sorted(range(len(data)), key=lambda i: -int(data[i][j]))[:top]
        for i in idx:
            print(f"  {int(data[i][j]):5d} {data[i][ia][-5:]} {data[i][isrc].strip()[:70]}")
            for k in range(max(0, i - ctx), i):
                print(f"        {data[k][ia][-5:]} {data[k][isrc].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
