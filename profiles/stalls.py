"""Per-kernel stall summary from an ncu report's source page.

    python profiles/stalls.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys
from collections import Counter

NAMES = ['stall_barrier', 'stall_branch_resolving', 'stall_dispatch', 'stall_lg', 'stall_long_sb',
         'stall_math', 'stall_mio', 'stall_no_inst', 'stall_not_selected', 'stall_selected',
         'stall_short_sb', 'stall_wait']


def num(x):
    try:
        return int(x or 0)
    except ValueError:
        return 0


def main(rep, kernel=None, top=12):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["--kernel-name", "regex:" + kernel]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    # a report with several launches repeats the table: keep the first one
    data = []
    for r in rows[2:]:
        if len(r) != len(hdr) or r[0] == hdr[0]:
            if data:
                break
            continue
        data.append(r)
    idx = {n: hdr.index(n) for n in NAMES}
    isrc = hdr.index('Source')
    iall = hdr.index('Warp Stall Sampling (All Samples)')
    tot = sum(num(r[iall]) for r in data)
    print("samples", tot)
    print(" ".join("%s=%.1f%%" % (n[6:], 100 * sum(num(r[idx[n]]) for r in data) / max(tot, 1))
                   for n in NAMES))
    ops = Counter()
    for r in data:
        t = r[isrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith('@') else t[0]
        ops[op.split('.')[0]] += 1
    print("sass op counts:", ", ".join("%s:%d" % kv for kv in ops.most_common(14)))
    for r in sorted(data, key=lambda r: -num(r[iall]))[:top]:
        worst = max(NAMES, key=lambda n: num(r[idx[n]]))
        print("%5s %-14s %s" % (r[iall], worst[6:], r[isrc][:70]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
