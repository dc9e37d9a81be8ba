"""Run a few 3D stages (for ncu): python tools/prof3d.py N prec n steps"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dginputs  # noqa: E402
from paper_1304_5546_b200 import dg3  # noqa: E402
N, prec, n, steps = (int(a) for a in sys.argv[1:5])
VX, VY, VZ, E = dginputs.cube_tet_mesh(n)
c = dg3.dg3_setup(N, VX, VY, VZ, E, precision=prec)
x, y, z = c.nodes()
c.set_fields(*dginputs.cube_cavity_mode(x, y, z, 0.0))
c.run(dginputs.cfl_dt_3d(VX, VY, VZ, E, N), steps)
c.sync()
print("done")
