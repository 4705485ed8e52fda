"""Text summary of an `ncu --set full` report (every kernel in it).

    python profiles/summarize_ncu.py gpurun_out/x.ncu-rep > profiles/r01/x.txt
"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def main(rep):
    h, u, vs = raw(rep)
    for v in vs:
        if len(v) != len(h):
            continue
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("kernel:", name)
        for k in WANT:
            if k in h:
                i = h.index(k)
                print("  %-70s %s %s" % (k, v[i], u[i]))
        sys.stdout.flush()
        kid = v[h.index("Kernel Name")].split("(")[0].split("<")[0].split()[-1] \
            if "Kernel Name" in h else None
        subprocess.run([sys.executable, __file__.replace("summarize_ncu.py", "stalls.py"), rep]
                       + ([kid] if kid else []))


if __name__ == "__main__":
    main(sys.argv[1])
