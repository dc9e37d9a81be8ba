for N in 6 7 8 9; do
python - <<PY
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import dginputs
from paper_1304_5546_b200 import dg
N = $N
VX, VY, E = dginputs.rect_mesh(362)
dt = dginputs.cfl_dt(VX, VY, E, N)
for kv in (0, 1):
    c = dg.dg_setup(N, VX, VY, E, precision=4, kernel_variant=kv)
    x, y = c.nodes(); c.set_fields(*dginputs.cavity_mode(x, y, dginputs.C4_T0)); c.run(dt, 3); c.sync()
    s = torch.cuda.ExternalStream(c.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for r in range(3):
        e0.record(s); c.run(dt, 10); e1.record(s); e1.synchronize(); best = min(best, e0.elapsed_time(e1) / 50)
    print(N, "tcgen05" if kv else "tuned", round(best, 5)); c.destroy()
PY
done
