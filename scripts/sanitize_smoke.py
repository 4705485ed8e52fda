"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the library once — on-chip field + cluster step
(c0 exact and fast, N=4096 with TMEM twiddles), the large-N path (pass A,
TMA column pass, bookkeeping kernels) in both modes, transforms, atoms,
error traces, the direct engine, and the NCCL-captured sharded loop."""
import os
import socket
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, ".")
warnings.simplefilter("ignore")
from paper_1711_08604_b200 import core, distributed, engine, workloads as W  # noqa: E402

torch.cuda.set_device(0)
w = W.CONFIGS["c0"]
g0 = W.signal_for("c0")
grid0 = core.ParameterGrid(W.radii_for(w.m), w.n)
for eng in ("fft", "fft-fast", "direct"):
    d = core.decompose(g0, grid0, max_terms=4, engine=eng, dc_first=eng == "fft")
    print(eng, [s.point.angle_index for s in d.steps], flush=True)
core.error_trace(d, g0)
core.kernel_samples(0.3 + 0.2j, 1024)
n = 4096
g1 = W.pole_sum(n, 16, 0.9, 5)
grid1 = core.ParameterGrid(tuple(i / 64 for i in range(64)), n)
for eng in ("fft", "fft-fast"):
    d = core.decompose(g1, grid1, max_terms=3, engine=eng)
    print(eng, n, [s.point.angle_index for s in d.steps], flush=True)
nb = 1 << 16
g2 = W.pole_sum(nb, 16, 0.97, 6)
grid2 = core.ParameterGrid(tuple(0.99 * i / 5 for i in range(6)), nb)
for eng in ("fft", "fft-fast"):
    d = core.decompose(g2, grid2, max_terms=2, engine=eng, dc_first=True)
    print(eng, nb, [s.point.angle_index for s in d.steps], flush=True)
core.analytic_projection(g2.real)
s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
import torch.distributed as dist  # noqa: E402
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % port, rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
d = distributed.decompose_sharded(g0, grid0, max_terms=3)[0]
print("sharded", [s.point.angle_index for s in d.steps], flush=True)
dist.destroy_process_group()
torch.cuda.synchronize()
print("sanitize smoke done")
