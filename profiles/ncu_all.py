"""Key metrics of every kernel in an `ncu --set full` report (one block each).

    python profiles/ncu_all.py gpurun_out/x.ncu-rep > profiles/r02/x.txt
"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from summarize_ncu import WANT  # noqa: E402

EXTRA = [
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_not_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_dispatch_stall_per_warp_active.pct",
    "smsp__warp_issue_stalled_membar_per_warp_active.pct",
    "smsp__warp_issue_stalled_sleeping_per_warp_active.pct",
]


def main(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    name_i = head.index("Kernel Name")
    for r in rows[2:]:
        print("kernel:", r[name_i][:150])
        for key in WANT + EXTRA:
            if key in head:
                i = head.index(key)
                print("  %-70s %s %s" % (key, r[i], units[i]))
        print()


if __name__ == "__main__":
    main(sys.argv[1])
