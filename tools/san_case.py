"""Small runs of every stage-kernel family for compute-sanitizer (tools/sanitize.sh): C1 (N=4 fp64),
the multi-tile persistent pipeline (grid capped: each CTA walks several tiles) for the S=1 fp32
3xTF32 (N=5), S=3 fp32 FMA (N=3), the fp64 DMMA unit teams (N=5 S=1, N=9 S=3) and warp-specialised
kernels (N=6, 7, 8: DMMA warps + flux warps, mbarrier hand-offs), fused and split, the tcgen05 variant
(N=5), a two-layer material case, and 3-partition group runs (tile lists + halo; N=5 and the
warp-specialised N=8)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import dginputs  # noqa: E402
from paper_1304_5546_b200 import dg  # noqa: E402


def run(N, prec, n=8, steps=3, **kw):
    VX, VY, E = dginputs.jittered_mesh(n, seed=N)
    eps = mu = None
    if kw.pop("material", False):
        eps, mu = dginputs.two_layer_material(VX, VY, E)
    c = dg.dg_setup(N, VX, VY, E, eps=eps, mu=mu, precision=prec, **kw)
    x, y = c.nodes()
    c.set_fields(*dginputs.cavity_mode(x, y, 0.1))
    c.run(dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu), steps)
    c.sync()
    f = c.get_fields()
    c.destroy()
    print(f"N={N} prec={prec} {kw}: ok, |Ez|max={np.abs(f[2]).max():.4f}", flush=True)


run(4, 8, n=16, steps=3)                                    # C1 shape
for fused in (True, False):
    run(5, 4, fused=fused, max_ctas=2)                      # 3xTF32 S=1, 4 tiles per CTA
    run(3, 4, fused=fused, max_ctas=2)                      # FMA S=3 split pipeline
    run(8, 8, fused=fused, max_ctas=2)                      # FMA fp64 S=3
    run(9, 8, fused=fused, max_ctas=2)                      # DMMA units S=3
    run(7, 8, fused=fused, max_ctas=2)                      # warp-specialised DMMA (fused), S=3 (split)
    run(5, 8, fused=fused, max_ctas=2)                      # DMMA units S=1
run(5, 4, n=12, max_ctas=1, kernel_variant=1)               # tcgen05, 3 groups per CTA
run(5, 4, n=12, max_ctas=1, kernel_variant=1, fused=False)
run(8, 8, material=True, max_ctas=2)                        # warp-specialised, material flux
run(6, 8, n=12, max_ctas=1)                                 # warp-specialised, one CTA walks every tile
VX, VY, E = dginputs.jittered_mesh(10, seed=3)
cs = [dg.dg_setup(5, VX, VY, E, precision=8, rank=r, nranks=3, transport=1, max_ctas=2) for r in range(3)]
for c in cs:
    x, y = c.nodes()
    c.set_fields(*dginputs.cavity_mode(x, y, 0.1))
dg.dg_run_group(cs, 1e-3, 3)
for c in cs:
    c.sync()
    c.destroy()
print("group ok")
cs = [dg.dg_setup(8, VX, VY, E, precision=8, rank=r, nranks=3, transport=1, max_ctas=2) for r in range(3)]
for c in cs:
    x, y = c.nodes()
    c.set_fields(*dginputs.cavity_mode(x, y, 0.1))
dg.dg_run_group(cs, 1e-4, 3)
for c in cs:
    c.sync()
    c.destroy()
print("group ws ok")
