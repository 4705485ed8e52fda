"""AFD grid-evaluation throughput on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

Workload (default; BASELINE.json configs[4], "c4", the largest configuration
and the one north_star sets its targets on): one analytic signal (128-pole
sum, |b| < 0.99, seeded), N = 2^20 samples, M = 16384 radii r_m = m/M,
20 AFD steps: 2^34 grid points per step.  A bench step is one full
decomposition (M*N*20 grid evals) with the input resident in HBM; `value` =
whole-job grid evals/s; `e2e` = the same through the public API
(`core.decompose`, host numpy in, host results out: pinned H2D + D2H inside
the timed region).  `--config c0..c3` selects the other BASELINE workloads
(parity cases; their lines are kept under profiles/).

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself
under `torch.distributed.run` with N ranks (one per GPU).  c4/c2 shard the
radius grid (one 32-byte candidate all-gather per AFD step), c3 shards the
signals, c0/c1 run replicas; time = max over ranks.

--impl reference times the reference's CPU implementation: the oracle port
(oracle/afd_oracle.c, a bit-exact C restatement of the reference; the
reference itself is pure Python and cannot travel to the GPU box) on all
host threads, on a bounded sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
warnings.simplefilter("ignore", UserWarning)

METRIC = "AFD grid evals/sec (M*N*steps/s)"
UNIT = "grid_evals/s"


def flops_per_eval(n):
    """F(N) = 5 log2 N + 7 FP64 flops per grid eval."""
    return 5 * (int(n).bit_length() - 1) + 7


def r_power_live(n, radii):
    """Live r^l entries per radius (distributed.live_powers)."""
    from paper_1711_08604_b200.distributed import live_powers
    return live_powers(radii, n)


def bytes_per_eval(n, radii=None):
    """Algorithmic HBM bytes per grid eval of the field: 0 for
    N <= 8192 (on-chip transform, the r^l table and spectrum stay in L2); for
    larger N the row-batch intermediate is written and read once (32 B) and
    the r^l table no longer fits in L2: 8 B per entry that is not an exact
    zero of the fold (those are never loaded, `r_power_live`)."""
    if n <= 8192:
        return 0.0
    if radii is None:
        return 40.0
    return 32.0 + 8.0 * float(r_power_live(n, radii).sum()) / (len(radii) * n)


def hbm_peak_gbs():
    """MEASURED_PEAKS.json (driver-written) else the profiling guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def fp64_instr_per_eval(n):
    """FP64-pipe instructions per grid eval of the exact field kernel: prologue
    2 DMUL, stage 0 2 DADD, each later stage 4 (2 DMUL + 2 DFMA + 4 DADD per
    butterfly) except the twiddle-index-0 butterflies of stages 1-3 (pass 0:
    1.75 per eval skipped), epilogue 2 DMUL scale + 3 for |.|^2 + 1 DSETP
    (DESIGN.md §4)."""
    k = int(n).bit_length() - 1
    return 2 + 2 + 4 * (k - 1) - 1.75 + 6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--mode", default="fast", choices=["exact", "fast"],
                    help="exact: bit-identical to the reference; fast: FP64 radix-16/fused "
                         "butterflies, r^l on chip (identical indices, 1e-9 relative)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--e2e-reps", type=int, default=0)
    ap.add_argument("--shard", default="auto", choices=["auto", "replicas", "signals", "radii"],
                    help="multi-GPU mode (auto: c3 signals, c2/c4 radii, else replicas)")
    return ap.parse_args()


def maybe_spawn(args):
    """`--gpus N` (N > 1) outside torchrun: re-launch under torch.distributed.run
    with N ranks on this node (rendezvous on 127.0.0.1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(cfg):
    from paper_1711_08604_b200 import workloads as W
    w = W.CONFIGS[cfg]
    return w, W.radii_for(w.m)


def host_signals(w, cfg, project=None):
    from paper_1711_08604_b200 import workloads as W
    sig = np.stack([W.signal_for(cfg, i) for i in range(w.batch)])
    if w.real:
        sig = project(sig)
    return sig


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, ~200 Hz)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= fn(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on the host cores
# ---------------------------------------------------------------------------
CPU_SAMPLE_EVALS = 1 << 24  # grid evals per sampled AFD step on the CPU


def cpu_sample(w, radii):
    """The CPU legs' bounded sample: every radius up to 2^24 grid evals per AFD
    step (c0, c1, c3), else an evenly strided subset of the radii and one AFD
    step (c2: 256 of 4096 radii, c4: 16 of 16384) — the oracle's cost per eval
    does not depend on which radii."""
    stride = max(1, -(-w.m * w.n // CPU_SAMPLE_EVALS))
    r = np.array(radii)[::stride]
    return r, (w.steps if stride == 1 else 1), stride


def cpu_baseline(w, radii, g, seconds):
    import oracle as O
    threads = O.max_threads()
    r, steps, stride = cpu_sample(w, radii)
    O.decompose(g, r, max_terms=1, threads=threads)  # warm tables / pages
    t0 = time.perf_counter()
    reps = 0
    while True:
        O.decompose(g, r, max_terms=steps, threads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds or reps >= 1000:
            break
    value = len(r) * w.n * steps * reps / el
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "%d x oracle decompose of %s signal 0 (%d AFD steps of M=%d%s x N=%d) "
                      "in %.1f s on %d threads"
                      % (reps, w.name, steps, len(r),
                         "" if stride == 1 else " (every %d-th of %d radii)" % (stride, w.m),
                         w.n, el, threads)}


def numpy_baseline(w, radii, g, seconds):
    """The reference's own numpy selection step (oracle/numpy_port.py: the
    cumprod tables, bit-reversed gather, stage loop, scale and first argmax of
    transform.py:73-93,137-201 and core.py:285-300 — the same bits as the
    reference) on one core, on the same radius sample as cpu_baseline: the
    reference package itself is not on the GPU box.  The tables are built
    once (the reference caches them per grid) and not timed."""
    import oracle as O
    from oracle import numpy_port as NP
    r, _, stride = cpu_sample(w, radii)
    t = NP.Tables(r, w.n)
    c = O.dft_forward(g)
    NP.select(t, c)
    t0 = time.perf_counter()
    reps = 0
    while True:
        NP.select(t, c)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds or reps >= 1000:
            break
    return {"value": len(r) * w.n * reps / el, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": "%d x the reference's numpy field + argmax (oracle/numpy_port.py, "
                      "bit-identical to the C oracle) for %s signal 0: M=%d%s x N=%d, "
                      "%.1f s on one core" % (reps, w.name, len(r),
                                               "" if stride == 1 else
                                               " (every %d-th of %d radii)" % (stride, w.m),
                                               w.n, el)}


# ---------------------------------------------------------------------------
# shared pieces of both arms
# ---------------------------------------------------------------------------
def shard_mode(args, w, world):
    """Multi-GPU mode of the workload: radius sharding for the
    single huge signals (c2, c4), signal sharding for the batch (c3),
    replicas for the small configs (c0, c1); 'single' on one GPU."""
    if args.shard != "auto":
        return args.shard
    if world == 1:
        return "single"
    return {"c3": "signals", "c2": "radii", "c4": "radii"}.get(w.name, "replicas")


def config_dict(args, w, world):
    """The `config` object of the JSON line — identical for both arms."""
    mode = shard_mode(args, w, world)
    par = {"single": "single", "replicas": "replicas x%d" % world}.get(
        mode, "dp%d over %s" % (world, mode))
    return {"workload": w.name, "n": w.n, "m": w.m, "afd_steps": w.steps, "signals": w.batch,
            "radii": "r_m = m/M", "parallelism": par,
            "l2": "flushed (512 MiB write) between timed iterations",
            "mode": ("exact (bit-identical to reference)" if args.mode == "exact" else
                     "fast (FP64 fused butterflies, r^l on chip; identical indices, 1e-9)")}


def scaling_of(mode):
    return "strong" if mode in ("radii", "signals") else "weak"


def check_parity(w, radii, sig0, rec0, count0, exact):
    """Signal 0 of the benchmarked output against the CPU oracle: the whole
    decomposition where the oracle finishes in seconds (<= 2^31 grid evals),
    else a replay of the GPU's selections (oracle.replay_check: the selected
    row's first maximum, neighbouring and sampled rows, coefficient and
    residual of every step).  exact: bitwise; fast: identical
    indices, 1e-9 relative."""
    import oracle as O
    rtol = 0.0 if exact else 1e-9
    radii = np.array(radii)
    t0 = time.perf_counter()
    if w.m * w.n * w.steps <= (1 << 31):
        o = O.decompose(sig0, radii, max_terms=w.steps)
        c = min(int(count0), w.steps)
        ok = c == len(o.steps) and np.array_equal(rec0["j"][:c], o.steps["j"]) and \
            np.array_equal(rec0["radius"][:c], o.steps["radius"])
        for key in ("c_re", "c_im", "residual"):
            a, b = rec0[key][:c], o.steps[key]
            ok = ok and (np.array_equal(a, b) if exact else
                         bool(np.all(np.abs(a - b) <= rtol * np.maximum(np.abs(b), 1e-300))))
        return {"ok": bool(ok), "method": "full oracle decomposition of signal 0 (%d steps)" % c,
                "seconds": round(time.perf_counter() - t0, 1)}
    r = O.replay_check(sig0, radii, rec0, int(count0), rows_per_step=6, rtol=rtol,
                       threads=O.max_threads())
    ok = r["ok"] and int(count0) == w.steps
    return {"ok": bool(ok), "method": "oracle replay of the GPU's %d selections: selected row, "
            "rows s+-2, last row and 6 seeded rows per step (%d rows of %d-point field in total)"
            % (int(count0), r["rows"], w.n), "why": r["why"],
            "seconds": round(time.perf_counter() - t0, 1)}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    w, radii = workload(args.config)
    g = host_signals(w, args.config, project=lambda s: np.stack([O.analytic_projection(x.real)
                                                                  for x in s]))[0]
    r, max_afd, stride = cpu_sample(w, radii)
    threads = O.max_threads()
    # size the sample: one AFD step costs t1; budget ~90 s for warmup + steps
    t0 = time.perf_counter()
    O.decompose(g, r, max_terms=1, threads=threads)
    t1 = time.perf_counter() - t0
    budget = 90.0 / max(1, args.steps + args.warmup)
    afd = int(max(1, min(max_afd, budget // max(t1, 1e-6))))
    for _ in range(args.warmup):
        O.decompose(g, r, max_terms=afd, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.decompose(g, r, max_terms=afd, threads=threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    evals = len(r) * w.n * afd  # one signal
    value = evals * args.steps / total
    sample = ("oracle port (bit-exact C restatement of the reference) decomposing %s signal 0: "
              "first %d of %d AFD steps (M=%d%s, N=%d) per bench step, %d threads"
              % (w.name, afd, w.steps, len(r),
                 "" if stride == 1 else " of %d radii, every %d-th" % (w.m, stride), w.n, threads))
    mode = shard_mode(args, w, world)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": scaling_of(mode), "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded BASELINE generator, SURVEY.md §8(d))",
        "impl": "reference", "config": config_dict(args, w, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def field_roofline(plan, w, radii_rows, ghat, exact, local):
    """Roofline of the field (the dominant kernel): CUDA-event launch time of
    one field evaluation over the plan's rows for `ghat` (on this stream),
    against FP64 (N <= 8192) or HBM (large N: the row-batch intermediate and,
    in exact mode, the live r^l table)."""
    from paper_1711_08604_b200 import engine
    rows = len(radii_rows)
    batch = ghat.shape[0]
    plan.time_field(ghat, reps=2)
    field_ms = plan.time_field(ghat, reps=5 if w.n > 8192 else 50)
    fpe = flops_per_eval(w.n)
    launch_evals = batch * rows * w.n
    bpe = bytes_per_eval(w.n, radii_rows) if exact else (32.0 if w.n > 8192 else 0.0)
    split = None
    tiers = plan.field_tier_rows() if not exact else {}
    if len(tiers) > 1:
        # pruned fast field (afd_pruned.cuh): a row whose weight tail beyond
        # l = L is negligible is evaluated from its first L spectrum terms —
        # in registers (L = 32, 64, 128) or as on-chip L-point transforms of
        # pre-twiddled spectra (L = 1024, 4096): F(L) flops, no HBM bytes (the
        # spectra and the weight tables are L2-resident).  The rest: large N
        # the two-pass path (F(N) flops, 32 B per eval); on-chip N (batches,
        # rows summed over the signals) the N-point field kernel, F(N) flops.
        big = w.n > 8192
        full = tiers.pop(w.n, 0)
        total = float(sum(tiers.values()) + full)
        fpe = (sum(r * flops_per_eval(t) for t, r in tiers.items()) + full * fpe) / total
        bpe = 32.0 * full / total if big else 0.0
        split = {"rows_%d" % t: r for t, r in tiers.items()}
        split.update({"flops_per_eval_%d" % t: flops_per_eval(t) for t in tiers})
        if big:
            split.update({"onchip_rows": sum(tiers.values()), "twopass_rows": full,
                          "flops_per_eval_twopass": flops_per_eval(w.n),
                          "bytes_per_eval_twopass": 32.0})
        else:
            split.update({"rows_%d" % w.n: full, "flops_per_eval_%d" % w.n: flops_per_eval(w.n),
                          "rows_are": "summed over the batch's signals"})
        split["note"] = ("rows whose weight tail beyond l = L is below 2^-64 of the largest kept "
                         "term are evaluated from their first L spectrum terms: L = 32, 64, 128 "
                         "in registers (one thread per 32 outputs), L = 1024, 4096 as N/L "
                         "on-chip L-point fields; credited F(L) = 5 log2 L + 7 flops per eval "
                         "(DESIGN.md §4)")
    achieved = launch_evals * fpe / (field_ms * 1e-3) / 1e12
    peak = engine.fp64_peak_tflops(local)
    hbm_peak, hbm_src = hbm_peak_gbs()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("field_%s_%s" % (
            "exact" if exact else "fast", w.name))
    instr = fp64_instr_per_eval(w.n) if exact else None
    fp64 = {"achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_source": "builder-measured in-run DFMA microbenchmark (afd_fp64_peak); "
                           "MEASURED_PEAKS.json has no FP64 entry"}
    if bpe and launch_evals * bpe / (hbm_peak * 1e9) > launch_evals * fpe / (peak * 1e12):
        hbm = launch_evals * bpe / (field_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": hbm, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm / hbm_peak, "traffic": traffic, "bytes_per_eval": bpe,
                "peak_source": hbm_src, "fp64": fp64}
    else:
        roof = dict(fp64, bound="fp64", traffic=traffic, bytes_per_eval=bpe)
        if instr:
            # bit-exact radix-2 arithmetic is mostly unfused: per eval the
            # kernel issues `instr` FP64-pipe instructions for F(N) flops
            roof["fp64_instr_per_eval"] = instr
            roof["frac_ceiling_at_this_instruction_mix"] = fpe / (2.0 * instr)
    roof.update({
        "kernel": ("field_kernel (fused prologue + inverse DIT + scale + |.|^2 + argmax)"
                   if w.n <= 8192 and split is None else
                   "batched pruned field: register tiers (field_reg_kernel<1>, <2>, <4>, BATCH) + "
                   "N-point rows (field_kernel)" if w.n <= 8192 else
                   "large-N field: pass A (big_field_a) + TMA column pass (col_tma_kernel)"
                   if split is None else
                   "pruned large-N field: register tiers (field_reg_kernel<1>, <2>, <4>), on-chip "
                   "256- ... 4096-point fields (field_sub_kernel<8>, <9>, field_warp_kernel, "
                   "field_kernel<12>) + two-pass rows (big_field_a + col_tma_kernel)"),
        "flops_per_eval": fpe, "evals_per_launch": launch_evals, "launch_ms": field_ms})
    if split is not None:
        roof["split"] = split
    return roof


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1711_08604_b200 import core, engine
    dev = torch.device("cuda", local)
    w, radii = workload(args.config)
    exact = args.mode == "exact"
    fast = 0 if exact else 1

    def project(sig):
        p = engine.get_plan((0.0,), w.n, batch=len(sig))
        return p.analytic_projection(torch.from_numpy(sig.astype(np.complex128)).to(dev)) \
            .cpu().numpy()

    sig = host_signals(w, args.config, project=project)
    mode = shard_mode(args, w, world)
    if mode in ("signals", "radii"):
        return run_sharded(args, w, radii, sig, mode, world, rank, local, dev)
    plan = engine.get_plan(radii, w.n, batch=w.batch, fast=fast)
    g_dev = torch.from_numpy(sig).to(dev)
    out = plan.alloc_outputs(w.batch, w.steps)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        plan.decompose(g_dev, w.steps, out=out)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    l0 = plan.launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush between timed iterations (not timed)
            ev[i][0].record(stream)
            plan.decompose(g_dev, w.steps, out=out)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = plan.launch_count() - l0
    barrier()
    torch.cuda.synchronize()
    total_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    evals = w.batch * w.m * w.n * w.steps
    value = world * evals * args.steps / (total_ms * 1e-3)
    step_ms = total_ms / args.steps

    recs, counts = out.host_steps()
    parity = None
    if not args.no_parity and rank == 0:
        parity = check_parity(w, radii, sig[0], recs[0], counts[0], exact)

    ghat = plan.dft_forward(g_dev)
    roofline = field_roofline(plan, w, radii, ghat, exact, local)
    if exact and w.n <= 8192 and w.batch * w.m < 16384:
        # the same kernel with enough rows to fill the GPU many times over
        # (c3's regime: 128 spectra x 1024 radii r_m = m/1024): the small
        # workloads' own launch is two rows per row-group, latency-bound
        sb, sm_ = 128, 1024
        splan = engine.Plan(tuple(m / sm_ for m in range(sm_)), w.n, max_batch=sb,
                            device=local, fast=fast)
        rng = np.random.default_rng(5)
        sx = torch.from_numpy(rng.standard_normal((sb, w.n)) +
                              1j * rng.standard_normal((sb, w.n))).to(dev)
        sgh = splan.dft_forward(sx)
        splan.time_field(sgh, reps=2)
        sms = splan.time_field(sgh, reps=10)
        fpe = flops_per_eval(w.n)
        sach = sb * sm_ * w.n * fpe / (sms * 1e-3) / 1e12
        roofline["steady_state"] = {
            "evals_per_launch": sb * sm_ * w.n, "launch_ms": sms, "achieved": sach,
            "frac": sach / roofline["peak"],
            "note": "same field kernel at N=%d, %d signals x M=%d radii" % (w.n, sb, sm_)}
        del splan, sx, sgh
    roofline["field_share_of_step"] = roofline["launch_ms"] * w.steps / step_ms

    # e2e through the public API, host buffers, pinned H2D + D2H in the region
    grid = core.ParameterGrid(radii, w.n)
    engine_name = "fft" if exact else "fft-fast"
    e2e_reps = args.e2e_reps or max(2, min(args.steps, int(20e3 / max(step_ms, 1e-3))))
    plan.decompose_host(sig, w.steps)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_reps):
        if w.batch == 1:
            core.decompose(sig[0], grid, max_terms=w.steps, engine=engine_name)
        else:
            core.decompose_batch(sig, grid, max_terms=w.steps, engine=engine_name)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    _, _, _, _, h2d, d2h = plan.decompose_host(sig, w.steps)
    e2e = {"value": world * evals * e2e_reps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "reps": e2e_reps,
           "api": "paper_1711_08604_b200.core.decompose%s(engine=%r)"
                  % ("" if w.batch == 1 else "_batch", engine_name)}

    cpu = cpu_np = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, radii, sig[0], args.cpu_seconds)
        cpu_np = numpy_baseline(w, radii, sig[0], args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": scaling_of(mode), "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded BASELINE generator, SURVEY.md §8(d))",
            "config": config_dict(args, w, world),
            "gpu_launches": launches,
            "parity_vs_oracle": None if parity is None else parity["ok"],
            "parity": parity,
            "roofline": roofline,
            "e2e": e2e,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "cpu_baseline_numpy": cpu_np,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(args, w, radii, sig, mode, world, rank, local, dev):
    """Strong-scaling multi-GPU modes: `signals` (each rank decomposes its
    block of the batch, no collective) and `radii` (each rank owns a block of
    the radius grid; per step one 32-byte candidate all-gather over NCCL,
    then every rank applies the same update: distributed.py)."""
    import torch
    import torch.distributed as dist
    from paper_1711_08604_b200 import core, distributed as D, engine

    exact = args.mode == "exact"
    fast = 0 if exact else 1
    if not dist.is_initialized():  # explicit --shard on one GPU without torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    lo, hi = 0, w.batch
    if mode == "signals":
        lo, hi = D.shard_bounds(w.batch, rank, world)
        m0, m1, b = 0, w.m, hi - lo
        plan = engine.get_plan(radii, w.n, batch=max(b, 1), fast=fast)
        g_dev = torch.from_numpy(sig[lo:hi]).to(dev)
        out = plan.alloc_outputs(max(b, 1), w.steps)

        def run():
            if b > 0:
                plan.decompose(g_dev, w.steps, out=out)

        def records():
            recs, counts = out.host_steps()
            return recs[0], int(counts[0])
    else:
        m0, m1 = D.radius_shard_bounds(radii, w.n, rank, world, exact=exact)
        b = w.batch
        plan = engine.get_plan(radii, w.n, batch=b, m0=m0, m1=m1, fast=fast)
        g_dev = torch.from_numpy(sig).to(dev)
        runner = D.ShardedRunner(plan, b, w.steps, None, False, group=None)

        def run():
            runner.run(g_dev)

        def records():
            rec, counts = runner.host_records()
            return rec[0], int(counts[0])

    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    l0 = plan.launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            run()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = plan.launch_count() - l0
    dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([float(sum(a.elapsed_time(bb) for a, bb in ev))], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    evals = w.batch * w.m * w.n * w.steps
    value = evals * args.steps / (total_ms * 1e-3)
    step_ms = total_ms / args.steps

    parity = None
    if rank == 0 and not args.no_parity and (mode == "radii" or hi > lo):
        rec, count = records()
        parity = check_parity(w, radii, sig[lo], rec, count, exact)

    # roofline of this rank's field launches (its rows, one signal)
    gh = plan.dft_forward(torch.from_numpy(sig[lo:lo + 1]).to(dev))
    roofline = field_roofline(plan, w, radii[m0:m1], gh, exact, local)
    roofline["field_share_of_step"] = roofline["launch_ms"] * w.steps * (
        1 if mode == "radii" else b) / step_ms

    # e2e through the public API with host buffers
    grid = core.ParameterGrid(radii, w.n)
    engine_name = "fft" if exact else "fft-fast"
    reps = args.e2e_reps or 2
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        if mode == "signals":
            if hi > lo:
                core.decompose_batch(sig[lo:hi], grid, max_terms=w.steps, engine=engine_name)
        else:
            D.decompose_sharded(sig, grid, max_terms=w.steps, engine_name=engine_name)
    torch.cuda.synchronize()
    tt = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = {"value": evals * reps / float(tt.item()), "unit": UNIT,
           "h2d_bytes_per_step": int(sig.nbytes if mode == "radii" else sig[lo:hi].nbytes),
           "d2h_bytes_per_step": int((sig.nbytes if mode == "radii" else sig[lo:hi].nbytes) +
                                     72 * w.steps * (b if mode == "signals" else w.batch)),
           "reps": reps,
           "api": ("paper_1711_08604_b200.core.decompose_batch" if mode == "signals" else
                   "paper_1711_08604_b200.distributed.decompose_sharded")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, SURVEY.md §8(d))",
            "config": config_dict(args, w, world),
            "gpu_launches": launches,
            "parity_vs_oracle": None if parity is None else parity["ok"], "parity": parity,
            "roofline": roofline, "e2e": e2e, "clocks": clk.summary(), "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    maybe_spawn(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
