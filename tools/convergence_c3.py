"""Config C3 (BASELINE.json configs[2]): h-refinement convergence at N=5 on the GPU, fp64,
K = 2,048 -> 524,288 (n = 32 .. 512), against the exact PEC-cavity mode (16, 16) after one
period T = 2 pi / omega (exact mode SPEC.md:431, pin P14).

    python tools/convergence_c3.py OUT.json

dt = O11 CFL estimate x min(1, (h / h0)^0.5) (h0 = 1/32), rounded down so that an integer number
of steps lands on T.  The error is the discrete L2 norm over all three fields,
||e|| = sqrt(2 dg_energy(e)) with e = q_gpu - q_exact at the nodes (dg_energy =
1/2 sum_k J_k e_k^T M e_k, mu = eps = 1): the library's own mass-matrix quadrature, no oracle.
Reported per mesh: error, observed order log2(e_{h} / e_{h/2}), ms per step (CUDA events),
DOF-updates/s -- accuracy against cost.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import dginputs  # noqa: E402
from paper_1304_5546_b200 import dg  # noqa: E402

N, MODE = 5, (16, 16)


def main():
    out = sys.argv[1]
    omega = math.pi * math.hypot(*MODE)
    T = 2 * math.pi / omega
    rows = []
    for n in (32, 64, 128, 256, 512):
        VX, VY, E = dginputs.rect_mesh(n)
        K = E.shape[0]
        dt0 = dginputs.cfl_dt(VX, VY, E, N) * min(1.0, math.sqrt(32.0 / n))
        steps = int(math.ceil(T / dt0))
        dt = T / steps
        c = dg.dg_setup(N, VX, VY, E, precision=8)
        x, y = c.nodes()
        c.set_fields(*dginputs.cavity_mode(x, y, 0.0, *MODE))
        c.run(dt, 1)
        c.sync()
        c.set_fields(*dginputs.cavity_mode(x, y, 0.0, *MODE))  # warm (graph captured), restart at t = 0
        s = torch.cuda.ExternalStream(c.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        c.run(dt, steps)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        c.sync()
        got = c.get_fields()
        ex = dginputs.cavity_mode(x, y, T, *MODE)
        c.set_fields(*(a - b for a, b in zip(got, ex)))
        err = math.sqrt(2.0 * c.energy())
        c.set_fields(*ex)
        norm = math.sqrt(2.0 * c.energy())
        maxerr = max(float(np.abs(a - b).max()) for a, b in zip(got, ex))
        c.destroy()
        Np = (N + 1) * (N + 2) // 2
        row = dict(n=n, K=K, h=1.0 / n, dt=dt, steps=steps, l2_error=err, l2_rel=err / norm, max_error=maxerr,
                   ms_per_step=ms / steps, dof_per_s=Np * K * 15 * steps / (ms * 1e-3))
        if rows:
            row["order"] = math.log2(rows[-1]["l2_error"] / err)
        rows.append(row)
        print(json.dumps(row), flush=True)
    with open(out, "w") as fh:
        json.dump(dict(_doc="C3 h-convergence, N=5 fp64, cavity mode (16,16), one period (tools/convergence_c3.py)",
                       T=T, rows=rows), fh, indent=1)


if __name__ == "__main__":
    main()
