"""Write tests/golden/pipeline_gate_n12.npz: the fp64 ORACLE (oracle/ only) after 100 LSERK4 steps
on the jittered 12x12 A16 mesh (K = 288: 9 tiles of 32 elements) for N = 1..9, constant material,
from the (1,1) cavity mode started so that it ends at phase pi/4 (dginputs.balanced_start, stored per N
as t0_<N>) + a seeded 1e-2 perturbation.

tools/tune.py gates every timed kernel variant on these fields (per-field A14 <= 1e-12 fp64 /
2e-5 fp32, run with dg_options.max_ctas = 2 so each CTA walks 4-5 tiles): "every
timed variant passes the oracle gate"; the paper's variant loop.

    python tools/make_pipeline_gate_golden.py     (~30 s, CPU only)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dginputs  # noqa: E402
from oracle.solver import Oracle  # noqa: E402

n, steps = 12, 100
VX, VY, E = dginputs.jittered_mesh(n, seed=12)
out = dict(n=n, steps=steps, amplitude=1e-2, VX=VX, VY=VY, EToV=E,
           doc="fp64 oracle fields after 100 LSERK4 steps, written by tools/make_pipeline_gate_golden.py")
for N in range(1, 10):
    o = Oracle(N, VX, VY, E)
    dt = dginputs.cfl_dt(VX, VY, E, N)
    t0 = dginputs.balanced_start(steps * dt)
    q0 = dginputs.cavity_mode(o.geo.x, o.geo.y, t0)
    q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(o.geo.x.shape, 1e-2, seed=N)))
    q = o.run(q0, dt, steps)
    out[f"dt{N}"] = dt
    out[f"t0_{N}"] = t0
    for nm, a in zip(("Hx", "Hy", "Ez"), q):
        out[f"{nm}{N}"] = a
    print(N, flush=True)
path = os.path.join(ROOT, "tests", "golden", "pipeline_gate_n12.npz")
np.savez_compressed(path, **out)
print("wrote", path)
