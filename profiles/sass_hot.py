"""Hottest SASS lines of one kernel from `ncu -i REP --page source --csv --print-source sass`.

    python profiles/sass_hot.py src.csv [top] [context]
Prints the top stall-sampled instructions in address order with their share.
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")

    def n(r):
        try:
            return int(r[i_s])
        except ValueError:
            return 0
    tot = sum(n(r) for r in data)
    print("total samples", tot, "instructions", len(data))
    best = sorted(range(len(data)), key=lambda k: -n(data[k]))[:top]
    for k in sorted(best):
        print("%5d %6d %5.1f%%  %s" % (k, n(data[k]), 100.0 * n(data[k]) / max(tot, 1),
                                       data[k][i_src].strip()[:100]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
