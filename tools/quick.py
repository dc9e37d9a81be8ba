"""Quick GPU check for kernel iteration: C4 throughput (fp32/fp64, fused) + N=5 parity vs oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import dginputs
from oracle.solver import Oracle
from paper_1304_5546_b200 import dg
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from probe import probe

N = int(os.environ.get("QN", "5"))
for prec in (4, 8):
    VX, VY, E = dginputs.rect_mesh(9)
    rng = np.random.default_rng(1)
    inner = (VX > 0) & (VX < 1) & (VY > 0) & (VY < 1)
    VX = VX + 0.25 / 9 * rng.uniform(-1, 1, VX.shape) * inner
    o = Oracle(N, VX, VY, E)
    q0 = tuple(a + b for a, b in zip(dginputs.cavity_mode(o.geo.x, o.geo.y, 0.0), dginputs.perturbation(o.geo.x.shape, 1e-2)))
    dt = dginputs.cfl_dt(VX, VY, o.EToV, N)
    want = o.run(q0, dt, 20)
    for fused in (True, False):
        c = dg.dg_setup(N, VX, VY, E, precision=prec, fused=fused)
        c.set_fields(*q0); c.run(dt, 20); got = c.get_fields()
        err = max(float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(got, want))
        c.set_fields(*q0)
        rerr = max(float(np.abs(a - b).max() / np.abs(b).max()) for a, b in zip(c.eval_rhs(0), o.rhs(q0)))
        print(f"parity N={N} prec={prec} fused={fused}: 20-step rel err {err:.2e}  rhs rel err {rerr:.2e}", flush=True)
        c.destroy()
for prec in (4, 8):
    probe(N, prec, 724 if N == 5 else 256, True)
