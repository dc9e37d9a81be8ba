"""Run a few stages of one configuration (for ncu): python tools/prof_one.py N prec n fused steps [variant]
(variant 1 = the fp32 tcgen05 kernels, dg_options.kernel_variant)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dginputs
from paper_1304_5546_b200 import dg
N, prec, n, fused, steps = (int(a) for a in sys.argv[1:6])
variant = int(sys.argv[6]) if len(sys.argv) > 6 else 0
VX, VY, E = dginputs.rect_mesh(n)
c = dg.dg_setup(N, VX, VY, E, precision=prec, fused=bool(fused), kernel_variant=variant)
x, y = c.nodes()
c.set_fields(*dginputs.cavity_mode(x, y, 0.0))
c.run(dginputs.cfl_dt(VX, VY, E, N), steps)
c.sync()
print("done")
