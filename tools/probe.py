"""Quick throughput probe: DOF-updates/s of dg_run for (N, prec, n, fused)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import dginputs
from paper_1304_5546_b200 import dg

def probe(N, prec, n, fused, steps=20):
    VX, VY, E = dginputs.rect_mesh(n)
    c = dg.dg_setup(N, VX, VY, E, precision=prec, fused=fused)
    x, y = c.nodes()
    q0 = dginputs.cavity_mode(x, y, 0.0)
    dt = dginputs.cfl_dt(VX, VY, E, N)
    c.set_fields(*q0)
    c.run(dt, 3); c.sync()
    c.profile(True)
    s = torch.cuda.ExternalStream(c.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); c.run(dt, steps); e1.record(s); e1.synchronize()
    ms = e0.elapsed_time(e1)
    st = c.kernel_stats()
    K = E.shape[0]; Np = (N+1)*(N+2)//2
    dofs = Np*K*3*5*steps
    ks = {k: (v['ms']/max(v['timed'],1)) for k, v in st.items() if v['timed']}
    print(f"N={N} prec={prec} K={K} fused={fused}: {ms/steps:.3f} ms/step  {dofs/(ms*1e-3)/1e9:.1f} GDOF/s  per-launch ms {ks}", flush=True)
    c.destroy()

if __name__ == "__main__":
    for N in range(1, 10):
        for prec in (4, 8):
            probe(N, prec, 181, True)
    for prec in (4, 8):
        probe(5, prec, 724, True)
        probe(5, prec, 724, False)
