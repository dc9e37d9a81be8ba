"""Diagnose the N=3 fp32 order-sweep case: determinism (3 runs bitwise), per-field error vs the oracle,
and where the largest error sits, for the tuned kernels and the tcgen05 variant."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import dginputs
from oracle.solver import Oracle
from paper_1304_5546_b200 import dg
N = int(sys.argv[1]) if len(sys.argv) > 1 else 3
VX, VY, E = dginputs.jittered_mesh(9, seed=N)
o = Oracle(N, VX, VY, E)
q0 = dginputs.cavity_mode(o.geo.x, o.geo.y, dginputs.C4_T0)
q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(o.geo.x.shape, 1e-2)))
dt = dginputs.cfl_dt(VX, VY, E, N)
for steps in (1, 10, 100):
    want = o.run(q0, dt, steps)
    for prec, var in ((4, 0), (4, 1), (8, 0)):
        runs = []
        for r in range(3):
            c = dg.dg_setup(N, VX, VY, E, precision=prec, kernel_variant=var)
            c.set_fields(*q0); c.run(dt, steps); runs.append(c.get_fields()); cfg = c.kernel_config(); c.destroy()
        det = all(np.array_equal(a, b) for r in runs[1:] for a, b in zip(r, runs[0]))
        errs = [float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(runs[0], want)]
        F = int(np.argmax(errs)); k, n = np.unravel_index(np.argmax(np.abs(runs[0][F] - want[F])), want[F].shape)
        print(f"steps={steps} prec={prec} {cfg['contraction']} S={cfg['slots']}: deterministic={det} per-field "
              f"{['%.2e' % x for x in errs]} worst field {F} elem {k} node {n} |want|={abs(want[F][k, n]):.3e} "
              f"max|F|={np.abs(want[F]).max():.3f}", flush=True)
