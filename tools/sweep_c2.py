"""Config C2 (BASELINE.json configs[1]): order sweep N=1..9 on the K=65,522-triangle cavity
(181x181 A16 mesh), fp32 and fp64, one B200, fused stage kernel and the split variant
(volume kernel vs surface+LIFT+RK kernel), each kernel against its own roofline.

    python tools/sweep_c2.py OUT.json [--steps S]

Per (N, precision, variant): DOF-updates/s over S graph-replayed LSERK4 steps (CUDA events on the
library's stream), then per-kernel launch times from the profiled graph replay (event-record nodes,
dg_profile), algorithmic bytes and flops per element-stage (bench.py's definitions), the fraction of
the measured HBM copy bandwidth and of the contraction pipe's measured peak.  Only the CUDA path
runs here (no oracle); inputs are the cavity mode (1,1), which the parity tests cover.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (algorithmic bytes / flops / peaks: one definition)
import dginputs  # noqa: E402
from paper_1304_5546_b200 import dg  # noqa: E402


def main():
    out = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 50
    n = 181
    VX, VY, E = dginputs.rect_mesh(n)
    K = E.shape[0]
    hbm, hbm_src = bench.peaks()
    rows = []
    for prec in (4, 8):
        for N in range(1, 10):
            Np = (N + 1) * (N + 2) // 2
            dt = dginputs.cfl_dt(VX, VY, E, N)
            for fused in (True, False):
                c = dg.dg_setup(N, VX, VY, E, precision=prec, fused=fused)
                x, y = c.nodes()
                c.set_fields(*dginputs.cavity_mode(x, y, 0.0))
                c.run(dt, 5)
                c.sync()
                s = torch.cuda.ExternalStream(c.stream())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                c.run(dt, steps)
                e1.record(s)
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                c.profile(True)
                c.run(dt, 10)
                st = c.kernel_stats()
                c.profile(False)
                kcfg = c.kernel_config()
                fin = bool(np.isfinite(c.get_fields()[2]).all())
                c.destroy()
                cb, cpeak, _ = bench.compute_peak(prec, kcfg["contraction"])
                row = dict(N=N, prec=prec, variant="fused" if fused else "split", K=K, steps=steps,
                           ms_per_step=ms / steps, dof_per_s=Np * K * 15 * steps / (ms * 1e-3),
                           contraction=kcfg["contraction"], finite=fin, kernels={})
                for kind in (("fused",) if fused else ("volume", "surface")):
                    k_ms = st[kind]["ms"] / (5 * 10)
                    by = bench.algorithmic_bytes_per_element_stage(Np, prec, kind) * K
                    fl = bench.flops_per_element_stage(N, kind) * K
                    row["kernels"][kind] = dict(
                        avg_launch_ms=k_ms, algorithmic_bytes=by, flops=fl,
                        hbm_gbs=by / (k_ms * 1e-3) / 1e9, hbm_frac=by / (k_ms * 1e-3) / 1e9 / hbm,
                        tflops=fl / (k_ms * 1e-3) / 1e12, compute_frac=fl / (k_ms * 1e-3) / 1e12 / cpeak,
                        compute_pipe=cb, intensity=fl / by, ridge=cpeak * 1e3 / hbm)
                rows.append(row)
                ks = " ".join(f"{k}:{v['avg_launch_ms']:.4f}ms hbm {v['hbm_frac']:.2f} cmp {v['compute_frac']:.2f}"
                              for k, v in row["kernels"].items())
                print(f"N={N} p={prec} {row['variant']:5s} {row['dof_per_s']:.3e} DOF/s  {ks}", flush=True)
    doc = ("C2 order sweep: 181x181 A16 cavity (K=65,522), N=1..9, fp32/fp64, fused and split, one B200 "
           "(tools/sweep_c2.py); peaks: HBM " + hbm_src + "; compute: bench.compute_peak")
    with open(out, "w") as fh:
        json.dump(dict(_doc=doc, hbm_gbs=hbm, rows=rows), fh, indent=1)


if __name__ == "__main__":
    main()
