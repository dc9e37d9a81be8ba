"""Write tests/golden/c4_oracle_100steps_sampled.npz: the fp64 ORACLE (oracle/ only) run on the
full config-C4 workload -- N=5, 724x724 A16 unit-square mesh (K=1,048,352), PEC cavity mode
(1,1) started at phase w t0 = pi/4 (so |H| ~ |Ez|: every field is O(1) and the per-field A14
quotient is well conditioned; DESIGN.md §2 A14) + seeded 1e-3 perturbation, dt = CFL estimate,
100 LSERK4 steps -- and the final fields sampled on a seeded set of elements (plus the per-field
global max |F| used by the A14 metric).

    python tools/make_c4_golden.py     (~30-60 min on 8 host cores; CPU only)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dginputs  # noqa: E402
from oracle.solver import Oracle  # noqa: E402

N, n, steps, nsample = 5, 724, 100, 4096
t0 = time.time()
VX, VY, E = dginputs.rect_mesh(n)
o = Oracle(N, VX, VY, E)
print(f"setup {time.time() - t0:.0f}s K={o.K}", flush=True)
q0 = dginputs.cavity_mode(o.geo.x, o.geo.y, dginputs.C4_T0)
q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(o.geo.x.shape, 1e-3)))
dt = dginputs.cfl_dt(VX, VY, E, N)
q = o.run(q0, dt, steps, callback=lambda s, q: print(f"step {s} {time.time() - t0:.0f}s", flush=True))
rng = np.random.default_rng(dginputs.SEED + 1)
elems = np.sort(rng.choice(o.K, nsample, replace=False))
elems = np.unique(np.concatenate([elems, [0, 1, o.K - 1, o.K - 2 * n]]))
out = os.path.join(ROOT, "tests", "golden", "c4_oracle_100steps_sampled.npz")
np.savez_compressed(out, N=N, n=n, steps=steps, dt=dt, t0=dginputs.C4_T0, seed=dginputs.SEED, amplitude=1e-3,
                    elements=elems, Hx=q[0][elems], Hy=q[1][elems], Ez=q[2][elems],
                    maxabs=np.array([np.abs(a).max() for a in q]),
                    doc="fp64 oracle, config C4 (SURVEY.md §8(d)), written by tools/make_c4_golden.py")
print("wrote", out, f"{time.time() - t0:.0f}s", flush=True)
