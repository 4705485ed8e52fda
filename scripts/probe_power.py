"""Sustained field throughput under the power cap:
    python scripts/probe_power.py N M FAST [SECONDS]

Runs back-to-back field evaluations for SECONDS (default 4) after a 1 s
warm-up, sampling NVML power, SM clock and throttle reasons every 10 ms;
prints ms per field (M rows), GB/s at 32 B/eval, mean power and median clock.
Short probes (probe_fast.py) finish before the power limiter reacts."""
import statistics
import sys
import threading
import time
import warnings

import numpy as np
import pynvml
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import engine, workloads as W  # noqa: E402

n, m, fast = (int(a) for a in sys.argv[1:4])
secs = float(sys.argv[4]) if len(sys.argv) > 4 else 4.0
plan = engine.Plan(W.radii_for(m), n, max_batch=1, fast=fast)
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((1, n)) + 1j * rng.standard_normal((1, n))).cuda()
gh = plan.dft_forward(x)
one = plan.time_field(gh, reps=1)
reps = max(1, int(0.25 / (one * 1e-3)))

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.01)


t_end = time.time() + 1.0
while time.time() < t_end:
    plan.time_field(gh, reps=reps)
th = threading.Thread(target=sampler, daemon=True)
th.start()
times = []
t_end = time.time() + secs
while time.time() < t_end:
    times.append(plan.time_field(gh, reps=reps))
stop.set()
th.join()
ms = statistics.median(times)
pw = statistics.mean(s[0] for s in samples)
clk = statistics.median(s[1] for s in samples)
reasons = 0
for s in samples:
    reasons |= s[2]
ev = m * n
print("N=%d M=%d fast=%d  field %.4f ms  %.0f GB/s at 32 B/eval  power %.0f W  sm %d MHz  "
      "reasons 0x%x  (%d samples)" % (n, m, fast, ms, ev * 32 / (ms * 1e-3) / 1e9, pw, clk,
                                      reasons, len(samples)), flush=True)
