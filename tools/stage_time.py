"""Time the fused stage kernel per (N, precision) on an n x n A16 mesh (graph replay, CUDA events).

    python tools/stage_time.py [--n 362] [--prec 4] [--orders 4,5,6] [--steps 20]

Prints one JSON line per order: ms per stage launch, DOF-updates/s, HBM fraction of the algorithmic
bytes (bench.algorithmic_bytes_per_element_stage) against MEASURED_PEAKS.json, kernel config."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import dginputs  # noqa: E402
from paper_1304_5546_b200 import dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=362)
ap.add_argument("--prec", type=int, default=4)
ap.add_argument("--orders", default="1,2,3,4,5,6,7,8,9")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
hbm, _ = bench.peaks()
VX, VY, E = dginputs.rect_mesh(a.n)
for N in [int(x) for x in a.orders.split(",")]:
    c = dg.dg_setup(N, VX, VY, E, precision=a.prec)
    x, y = c.nodes()
    c.set_fields(*dginputs.cavity_mode(x, y, dginputs.C4_T0))
    dt = dginputs.cfl_dt(VX, VY, E, N)
    c.run(dt, 5)
    c.sync()
    s = torch.cuda.ExternalStream(c.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    c.run(dt, a.steps)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (5 * a.steps)
    K, Np = c.K_local, c.Np
    ab = bench.algorithmic_bytes_per_element_stage(Np, a.prec) * K
    print(json.dumps(dict(N=N, prec=a.prec, n=a.n, K=K, ms_per_stage=round(ms, 5),
                          dof_per_s=Np * K * 3 / (ms * 1e-3), hbm_frac=ab / (ms * 1e-3) / 1e9 / hbm,
                          contraction=c.kernel_config()["contraction"])), flush=True)
    c.destroy()
