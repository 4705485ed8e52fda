"""AFD grid-evaluation throughput on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl reference]

Workload (BASELINE.json configs[1], "c1"): one analytic signal (32-pole sum,
|b| < 0.95, seeded), N = 4096 samples, M = 512 radii r_m = m/M, 30 AFD steps.
A bench step is one full decomposition (30 AFD steps = M*N*30 grid evals)
through the device-resident decomposition (CUDA graph of fused field+argmax
and step kernels, input resident in HBM).  `value` = whole-job grid evals/s;
`e2e` = the same through the public API `core.decompose` with the signal in
host memory (pinned H2D + D2H of the result inside the timed region).

Multi-GPU (torchrun, one rank per GPU): c1 does not shard (SURVEY.md §8(e):
"replicas only"); every rank decomposes its own replica, time = max over
ranks, value = all ranks' evals / that time, scaling "weak".

--impl reference times the reference's CPU implementation: the oracle port
(oracle/afd_oracle.c, a bit-exact C restatement of the reference; the
reference itself is pure Python and cannot travel to the GPU box) on all
host threads, on a bounded sample of the same workload.
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
    """Per radius, the first l with r^l == +0 in the reference's sequential fold
    (np.cumprod, transform.py:147-150), else n — the entries the large-N
    prologue must load.  Only r <= 0.5 ever reaches zero: for r > 0.5 the fold
    sticks at a subnormal (k * 2^-1074 * r rounds back to k * 2^-1074), so
    those rows are live to the end."""
    import numpy as np
    r = np.asarray(radii, dtype=np.float64)
    live = np.full(r.shape, n, dtype=np.int64)
    idx = np.nonzero(r <= 0.5)[0]
    v = np.ones(idx.size)
    rr = r[idx]
    for l in range(1, n):
        if idx.size == 0:
            break
        v = v * rr
        z = v == 0.0
        if z.any():
            live[idx[z]] = l
            keep = ~z
            idx, v, rr = idx[keep], v[keep], rr[keep]
    return live


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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--e2e-reps", type=int, default=0)
    ap.add_argument("--shard", default="auto", choices=["auto", "replicas", "signals", "radii"],
                    help="multi-GPU mode (auto: c3 signals, c2/c4 radii, else replicas)")
    return ap.parse_args()


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
              "first %d of %d AFD steps (M=%d%s, N=%d) per step, %d threads"
              % (w.name, afd, w.steps, len(r),
                 "" if stride == 1 else " of %d radii, every %d-th" % (w.m, stride), w.n, threads))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)", "impl": "reference",
        "config": {"workload": w.name, "n": w.n, "m": w.m, "afd_steps": w.steps,
                   "signals": w.batch, "sampled_afd_steps_per_bench_step": afd},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1711_08604_b200 import core, engine
    dev = torch.device("cuda", local)
    w, radii = workload(args.config)
    plan = engine.get_plan(radii, w.n, batch=w.batch)

    def project(sig):
        p = engine.get_plan((0.0,), w.n, batch=len(sig))
        return plan_to_np(p.analytic_projection(torch.from_numpy(sig.astype(np.complex128))
                                                .to(dev)))

    def plan_to_np(t):
        return t.cpu().numpy()

    sig = host_signals(w, args.config, project=project)
    # multi-GPU mode: replicas of the whole workload (c0/c1,
    # weak scaling), the signals of a batch split over the ranks (c3), or the
    # radius grid split over the ranks with one all-gather per step (c2/c4);
    # the last two are strong scaling.  One GPU: the single-plan path.
    mode = args.shard if args.shard != "auto" else {
        "c3": "signals", "c2": "radii", "c4": "radii"}.get(w.name, "replicas")
    if world == 1 and args.shard == "auto":
        mode = "single"
    if mode in ("signals", "radii"):
        return run_sharded(args, w, radii, sig, mode, world, rank, local, dev)
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
    per = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(per))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    evals = w.batch * w.m * w.n * w.steps
    value = world * evals * args.steps / (total_ms * 1e-3)

    # parity of the benchmarked output against the oracle (first signal;
    # for the big configs only the first `check` steps, replayed by the oracle)
    import oracle as O
    recs, counts = out.host_steps()
    check = w.steps if w.m * w.n * w.steps <= (1 << 31) else 2
    parity = None
    if not args.no_parity:
        o = O.decompose(sig[0], np.array(radii), max_terms=check)
        c = min(int(counts[0]), check)
        parity = bool(c == len(o.steps) and
                      np.array_equal(recs[0]["j"][:c], o.steps["j"]) and
                      np.array_equal(recs[0]["radius"][:c], o.steps["radius"]) and
                      np.array_equal(recs[0]["c_re"][:c], o.steps["c_re"]) and
                      np.array_equal(recs[0]["residual"][:c], o.steps["residual"]))

    # roofline: the fused field+argmax kernel, CUDA events on this stream
    ghat = plan.dft_forward(g_dev)
    plan.time_field(ghat, reps=5)
    field_ms = plan.time_field(ghat, reps=50)
    fpe = flops_per_eval(w.n)
    field_flops = w.batch * w.m * w.n * fpe
    achieved = field_flops / (field_ms * 1e-3) / 1e12
    peak = engine.fp64_peak_tflops(local)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("field_kernel_%s" % w.name)
    # the binding roofline: FP64 for N <= 8192 (0 algorithmic HBM bytes), HBM
    # for the large-N path (r^l table + row-batch intermediate)
    launch_evals = w.batch * w.m * w.n
    bpe = bytes_per_eval(w.n, radii)
    hbm_peak, hbm_src = hbm_peak_gbs()
    t_fp64 = launch_evals * fpe / (peak * 1e12)
    t_hbm = launch_evals * bpe / (hbm_peak * 1e9)
    if t_hbm > t_fp64:
        hbm_achieved = launch_evals * bpe / (field_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm_achieved / hbm_peak, "traffic": traffic,
                    "bytes_per_eval": bpe, "peak_source": hbm_src,
                    "fp64": {"achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": achieved / peak}}
    else:
        roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "peak_source": "measured in-run DFMA microbenchmark (afd_fp64_peak); "
                                   "MEASURED_PEAKS.json has no FP64 entry",
                    # bit-exact radix-2 arithmetic is mostly unfused: per eval the
                    # kernel issues fp64_instr_per_eval FP64-pipe instructions for
                    # F(N) flops, so even a saturated FP64 pipe reaches only this
                    # fraction of the DFMA peak
                    "fp64_instr_per_eval": fp64_instr_per_eval(w.n),
                    "frac_ceiling_at_this_instruction_mix":
                        fpe / (2.0 * fp64_instr_per_eval(w.n))}
        if w.batch * w.m < 16384:
            # the same kernel with enough rows to fill the GPU many times over
            # (c3's regime: 128 spectra x 1024 radii r_m = m/1024): the
            # workload's own launch is two rows per row-group, latency-bound
            sb, sm_ = 128, 1024
            # a private plan: the cached one keeps serving the e2e leg below
            splan = engine.Plan(tuple(m / sm_ for m in range(sm_)), w.n, max_batch=sb,
                                device=g_dev.device.index)
            rng = np.random.default_rng(5)
            sx = torch.from_numpy(rng.standard_normal((sb, w.n)) +
                                  1j * rng.standard_normal((sb, w.n))).to(g_dev.device)
            sgh = splan.dft_forward(sx)
            splan.time_field(sgh, reps=2)
            sms = splan.time_field(sgh, reps=10)
            sach = sb * sm_ * w.n * fpe / (sms * 1e-3) / 1e12
            roofline["steady_state"] = {
                "evals_per_launch": sb * sm_ * w.n, "launch_ms": sms, "achieved": sach,
                "frac": sach / peak,
                "note": "same field kernel at N=%d, %d signals x M=%d radii" % (w.n, sb, sm_)}
            del splan, sx, sgh
    roofline.update({
        "kernel": ("field_kernel (fused prologue + inverse DIT + scale + |.|^2 + argmax)"
                   if w.n <= 8192 else
                   "large-N field: big_pass_a + column pass(es) over the row batches"),
        "flops_per_eval": fpe, "evals_per_launch": launch_evals, "launch_ms": field_ms,
        "field_share_of_step": (field_ms * (w.steps) / (total_ms / args.steps))})

    # e2e through the public API, host buffers, pinned H2D + D2H in the region
    grid = core.ParameterGrid(radii, w.n)
    e2e_reps = args.e2e_reps or max(3, min(args.steps, 200))
    for _ in range(min(3, e2e_reps)):
        plan.decompose_host(sig, w.steps)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_reps):
        if w.batch == 1:
            core.decompose(sig[0], grid, max_terms=w.steps)
        else:
            core.decompose_batch(sig, grid, max_terms=w.steps)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    _, _, _, _, h2d, d2h = plan.decompose_host(sig, w.steps)
    e2e = {"value": world * evals * e2e_reps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "api": "paper_1711_08604_b200.core.decompose"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, radii, sig[0], args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, SURVEY.md §8(d))",
            "config": {"workload": w.name, "n": w.n, "m": w.m, "afd_steps": w.steps,
                       "signals": w.batch, "radii": "r_m = m/M",
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "flushed (512 MiB write) between timed iterations",
                       "mode": "exact (bit-identical to reference)"},
            "gpu_launches": launches,
            "parity_vs_oracle": parity,
            "roofline": roofline,
            "e2e": e2e,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
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
    from paper_1711_08604_b200 import _capi, core, distributed as D, engine

    if not dist.is_initialized():  # explicit --shard on one GPU without torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    if mode == "signals":
        lo, hi = D.shard_bounds(w.batch, rank, world)
        m0, m1, b = 0, w.m, hi - lo
        plan = engine.get_plan(radii, w.n, batch=max(b, 1))
        g_dev = torch.from_numpy(sig[lo:hi]).to(dev)
        out = plan.alloc_outputs(max(b, 1), w.steps)

        def run():
            if b > 0:
                plan.decompose(g_dev, w.steps, out=out)

        def records():
            recs, counts = out.host_steps()
            return recs[0], int(counts[0])
    else:
        m0, m1 = D.shard_bounds(w.m, rank, world)
        b = w.batch
        plan = engine.get_plan(radii, w.n, batch=b, m0=m0, m1=m1)
        g_dev = torch.from_numpy(sig).to(dev)
        steps_buf = torch.zeros((b, w.steps, _capi.STEP_DTYPE.itemsize), dtype=torch.uint8,
                                device=dev)
        gathered = torch.empty((world, b, 32), dtype=torch.uint8, device=dev)
        state = {}

        def run():
            plan.sharded_begin(g_dev)
            for k in range(w.steps):
                local_c = plan.select_local(k, False, b)
                dist.all_gather_into_tensor(gathered, local_c.contiguous())
                plan.apply_step(k, w.steps, None, False,
                                gathered.permute(1, 0, 2).contiguous(), steps_buf)
            state["fin"] = plan.sharded_finish(b)

        def records():
            rec = steps_buf.cpu().numpy().view(_capi.STEP_DTYPE)[..., 0]
            return rec[0], int(state["fin"][0].cpu().numpy()[0])

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

    import oracle as O
    parity = None
    if rank == 0 and not args.no_parity:
        rec, count = records()
        check = w.steps if w.m * w.n * w.steps <= (1 << 31) else 2
        o = O.decompose(sig[0], np.array(radii), max_terms=check)
        c = min(count, check)
        parity = bool(c == len(o.steps) and np.array_equal(rec["j"][:c], o.steps["j"]) and
                      np.array_equal(rec["radius"][:c], o.steps["radius"]) and
                      np.array_equal(rec["c_re"][:c], o.steps["c_re"]) and
                      np.array_equal(rec["residual"][:c], o.steps["residual"]))

    # roofline of this rank's field launches (its rows / signals)
    gh = plan.dft_forward(torch.from_numpy(sig[:1] if mode == "radii" else sig[lo:lo + 1])
                          .to(dev))
    plan.time_field(gh, reps=3)
    field_ms = plan.time_field(gh, reps=10)
    fpe = flops_per_eval(w.n)
    achieved = (m1 - m0) * w.n * fpe / (field_ms * 1e-3) / 1e12
    peak = engine.fp64_peak_tflops(local)
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "field_kernel / big_pass_a+big_pass_col (this rank's rows, one signal)",
                "flops_per_eval": fpe, "evals_per_launch": (m1 - m0) * w.n,
                "launch_ms": field_ms,
                "peak_source": "measured in-run DFMA microbenchmark (afd_fp64_peak)"}
    bpe = bytes_per_eval(w.n, radii[m0:m1])
    hbm_peak, hbm_src = hbm_peak_gbs()
    if bpe and bpe / (hbm_peak * 1e9) > fpe / (peak * 1e12):  # HBM-bound (large N)
        hbm = (m1 - m0) * w.n * bpe / (field_ms * 1e-3) / 1e9
        roofline.update({"bound": "hbm", "achieved": hbm, "peak": hbm_peak, "unit": "GB/s",
                         "frac": hbm / hbm_peak, "bytes_per_eval": bpe, "peak_source": hbm_src,
                         "fp64": {"achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                                  "frac": achieved / peak}})

    # e2e through the public API with host buffers
    grid = core.ParameterGrid(radii, w.n)
    reps = args.e2e_reps or 2
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        if mode == "signals":
            if hi > lo:
                core.decompose_batch(sig[lo:hi], grid, max_terms=w.steps)
        else:
            D.decompose_sharded(sig, grid, max_terms=w.steps)
    torch.cuda.synchronize()
    tt = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e = {"value": evals * reps / float(tt.item()), "unit": UNIT,
           "h2d_bytes_per_step": int(sig.nbytes if mode == "radii" else sig[lo:hi].nbytes),
           "d2h_bytes_per_step": None,
           "api": ("paper_1711_08604_b200.core.decompose_batch" if mode == "signals" else
                   "paper_1711_08604_b200.distributed.decompose_sharded")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, SURVEY.md §8(d))",
            "config": {"workload": w.name, "n": w.n, "m": w.m, "afd_steps": w.steps,
                       "signals": w.batch, "radii": "r_m = m/M",
                       "parallelism": "dp%d over %s" % (world, mode),
                       "l2": "flushed (512 MiB write) between timed iterations",
                       "mode": "exact (bit-identical to reference)"},
            "gpu_launches": launches, "parity_vs_oracle": parity, "roofline": roofline,
            "e2e": e2e, "clocks": clk.summary(), "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
