"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python profiles/launch_summary.py gpurun_out/launches.csv
Prints per-kernel launch counts, mean and total device time, and shares.
(ncu serialises launches and runs them cold, so compare shares, not
absolute step times.)
"""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    im = h.index("Metric Name") if "Metric Name" in h else None
    ig = h.index("Grid Size") if "Grid Size" in h else None
    agg = collections.defaultdict(list)
    dram = collections.defaultdict(float)
    for r in data:
        if len(r) <= iv:
            continue
        # launches of one kernel with different grids (e.g. the bench's
        # decomposition vs its saturated steady-state probe) listed apart
        name = r[ik].split("(")[0].replace("void ", "") + (" grid" + r[ig] if ig is not None else "")
        metric = r[im] if im is not None else "gpu__time_duration.sum"
        v = float(r[iv].replace(",", ""))
        if metric.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[iu], 1)
            dram[name] += v * scale
            continue
        if metric != "gpu__time_duration.sum":
            continue
        v = v / 1000 if r[iu] == "ns" else (v * 1000 if r[iu] == "ms" else v)
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        extra = "  dram %.3f GB" % (dram[k] / 1e9) if k in dram else ""
        out.append("%-86s n=%5d mean=%9.2f us total=%10.1f us share=%5.1f%%%s"
                   % (k[:86], len(v), sum(v) / len(v), sum(v), 100 * sum(v) / tot, extra))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
