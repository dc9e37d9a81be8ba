"""Run a few stages of a two-layer-material configuration (for ncu): python tools/prof_mat.py N prec n steps"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dginputs
from paper_1304_5546_b200 import dg
N, prec, n, steps = (int(a) for a in sys.argv[1:5])
VX, VY, E = dginputs.rect_mesh(n)
eps, mu = dginputs.two_layer_material(VX, VY, E)
c = dg.dg_setup(N, VX, VY, E, eps=eps, mu=mu, precision=prec)
x, y = c.nodes()
c.set_fields(*dginputs.cavity_mode(x, y, 0.0))
c.run(dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu), steps)
c.sync()
print("done")
