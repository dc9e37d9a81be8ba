"""Single-module kernel variants: the main libdg.so with ONE (N, precision) module rebuilt with other
knobs (every stage mode, so bench.py and the tests can run it through DG_LIB).

    python tools/modvar.py build TAG NAME=KNOBS ...   # CPU, e.g. N8_f64 R5_S3_C5_Y1=R:5,S:3,C:5,Y:1
    python tools/modvar.py time TAG OUT.jsonl [--n 362] [--mat] [--steps 20]   # GPU: every lib of TAG

Libraries go to build_modvar/<TAG>/<NAME>.so.  `time` runs each library in a fresh process: the fused
stage on an n x n A16 mesh (graph replay, CUDA events), and the per-field A14 oracle gate of tools/tune.py
(tests/golden/pipeline_gate_n12.npz, grid capped at 2 CTAs) for that (N, precision)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.environ.get("MODVAR_DIR") or os.path.join(ROOT, "build_modvar")


def build(tag, specs):
    from paper_1304_5546_b200 import build as B
    B.build()
    n = int(tag[1:tag.index("_")])
    ct = "float" if "_f32" in tag else "double"
    base = dict(B.tuning().get(tag, {}))
    if tag.endswith("_tc"):  # the tcgen05 variant module
        base = dict(B.TC_DEFAULT, **base, M=3, V=1)
    base.pop("ms", None)
    vdir = os.path.join(OUT, tag)
    os.makedirs(vdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v"] + B.ARCH
    inc = ["-I", B.CSRC, "-I", os.path.join(ROOT, "include")]
    main_objs = [os.path.join(B.BUILD, f"k_{t}.o") for t, _, _ in B.tags(B.NMAX_DEFAULT)]
    main_objs += [os.path.join(B.BUILD, f"k3_{t}.o") for t, _, _ in B.tags3()]
    main_objs += [os.path.join(B.BUILD, x) for x in ("setup3d.o", "runtime3d.o", "setup.o", "runtime.o")]
    import concurrent.futures as cf

    def one(spec):
        name, _, kv = spec.partition("=")
        knobs = dict(base)
        for item in filter(None, kv.split(",")):
            k, v = item.split(":")
            knobs[k] = int(v)
        src = os.path.join(vdir, f"k_{tag}_{name}.cu")
        B.write_if_changed(src, B.inst_source(tag, n, ct, knobs).replace(
            '#include "../kernels.cuh"', f'#include "{os.path.join(B.CSRC, "kernels.cuh")}"'))
        obj = src[:-3] + ".o"
        p = B.run([B.NVCC, "-c", src, "-o", obj] + common + inc)
        lines = (p.stdout + p.stderr).splitlines()
        regs = []
        for i, ln in enumerate(lines):  # the fused kernels: stage_kernel<0, false/true>
            if "Compiling entry function" in ln and ("stage_kernelILi0ELb" in ln or "stage_kernel_wsILi0ELb" in ln):
                info = " ".join(x.split(":", 1)[-1].strip() for x in lines[i + 1:i + 4] if "spill" in x or "registers" in x)
                regs.append(("ws " if "_ws" in ln else "") + ("mat " if "ILi0ELb1" in ln else "const ") + info)
        objs = [obj if o.endswith(f"k_{tag}.o") else o for o in main_objs]
        lib = os.path.join(vdir, f"{name}.so")
        B.run([B.NVCC, "-shared", "-o", lib] + objs + B.ARCH + ["-ldl"])
        return name, knobs, regs

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for name, knobs, regs in ex.map(one, specs):
            print(name, knobs, *regs[:2], sep="\n  ", flush=True)


CODE = r"""
import sys, json; sys.path.insert(0, @ROOT@)
import numpy as np, torch, dginputs
from paper_1304_5546_b200 import dg
N, PREC = @N@, @PREC@
VX, VY, E = dginputs.rect_mesh(@NN@)
dt = dginputs.cfl_dt(VX, VY, E, N)
kw = {}
if @MAT@:  # two-layer material (C5's recipe, dginputs.two_layer_material)
    eps, mu = dginputs.two_layer_material(VX, VY, E)
    kw = dict(eps=eps, mu=mu)
    dt = dginputs.cfl_dt(VX, VY, E, N, eps=eps, mu=mu)
c = dg.dg_setup(N, VX, VY, E, precision=PREC, kernel_variant=@KV@, **kw)
x, y = c.nodes()
c.set_fields(*dginputs.cavity_mode(x, y, dginputs.C4_T0))
c.run(dt, 3); c.sync()
s = torch.cuda.ExternalStream(c.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for rep in range(3):
    e0.record(s); c.run(dt, @STEPS@); e1.record(s); e1.synchronize()
    ms.append(e0.elapsed_time(e1) / (5 * @STEPS@))
cfg = c.kernel_config(); c.destroy()
G = np.load(@ROOT@ + "/tests/golden/pipeline_gate_n12.npz")
g = dg.dg_setup(N, G["VX"], G["VY"], G["EToV"], precision=PREC, max_ctas=2, kernel_variant=@KV@)
xg, yg = g.nodes()
q0 = dginputs.cavity_mode(xg, yg, float(G["t0_%d" % N]))
q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(xg.shape, float(G["amplitude"]), seed=N)))
g.set_fields(*q0); g.run(float(G["dt%d" % N]), int(G["steps"])); got = g.get_fields(); g.destroy()
gate = max(float(np.abs(a - G[nm + str(N)]).max() / np.abs(G[nm + str(N)]).max()) for a, nm in zip(got, ("Hx", "Hy", "Ez")))
print(json.dumps(dict(N=N, prec=PREC, n=@NN@, mat=bool(@MAT@), ms=min(ms), ms_all=ms, gate=gate, cfg=cfg)))
"""


def time_all(tag, out, n=362, mat=False, steps=20):
    N = int(tag[1:tag.index("_")])
    prec = 4 if "_f32" in tag else 8
    vdir = os.path.join(OUT, tag)
    libs = [("main", None)] + [(f[:-3], os.path.join(vdir, f)) for f in sorted(os.listdir(vdir)) if f.endswith(".so")]
    code = CODE
    for k, v in (("@ROOT@", repr(ROOT)), ("@NN@", str(n)), ("@N@", str(N)), ("@PREC@", str(prec)),
                 ("@MAT@", str(int(mat))), ("@STEPS@", str(steps)), ("@KV@", "1" if tag.endswith("_tc") else "0")):
        code = code.replace(k, v)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with open(out, "a") as fh:
        for name, lib in libs:
            env = dict(os.environ)
            if lib:
                env["DG_LIB"] = lib
            p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
            if p.returncode != 0:
                print(name, "FAILED", p.stderr[-800:], flush=True)
                continue
            r = json.loads(p.stdout.strip().splitlines()[-1])
            r["variant"] = name
            r["tag"] = tag
            fh.write(json.dumps(r) + "\n")
            print(f"{tag} {name:28s} {r['ms']:.5f} ms  gate {r['gate']:.2e}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "time":
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("tag")
        ap.add_argument("out")
        ap.add_argument("--n", type=int, default=362)
        ap.add_argument("--mat", action="store_true")
        ap.add_argument("--steps", type=int, default=20)
        a = ap.parse_args()
        time_all(a.tag, a.out, a.n, a.mat, a.steps)
