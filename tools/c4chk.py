import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import dginputs
from paper_1304_5546_b200 import dg
gold = np.load("tests/golden/c4_oracle_100steps_sampled.npz")
VX, VY, E = dginputs.rect_mesh(724)
c = dg.dg_setup(5, VX, VY, E, precision=int(os.environ.get("PREC", "4")))
x, y = c.nodes()
q0 = dginputs.cavity_mode(x, y, 0.0)
q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(x.shape, 1e-3)))
dt = float(gold["dt"]); print("dt match", dt == dginputs.cfl_dt(VX, VY, E, 5))
c.set_fields(*q0)
for s in (1, 10, 100):
    c.set_fields(*q0); c.run(dt, s); got = c.get_fields()
    if s == 100:
        el = gold["elements"]
        print(os.environ.get("DG_LIB", "main"), [float(np.abs(got[F][el] - gold[nm]).max() / gold["maxabs"][F]) for F, nm in enumerate(("Hx", "Hy", "Ez"))])
        ex = dginputs.cavity_mode(x, y, 100 * dt)
        print(" vs exact mode (global scale):", [float(np.abs(got[F] - ex[F]).max()) for F in range(3)])
        print(" gold vs exact mode:", [float(np.abs(gold[nm] - ex[F][el]).max()) for F, nm in enumerate(("Hx", "Hy", "Ez"))])
