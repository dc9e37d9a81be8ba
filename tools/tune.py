"""Autotuning of the stage-kernel knobs per (N, precision) -- the paper's
"looping over all variants and comparing timing data for each".

    python tools/tune.py build            # CPU: build one library per knob set -> build_variants/
    python tools/tune.py measure OUT.json # GPU: time the fused stage for every (variant, N, precision)
    python tools/tune.py pick OUT.json... # CPU: write paper_1304_5546_b200/csrc/tune.json
                                          #   (OUT.json:f64 = only that file's fp64 rows)

Knobs: R (max rows per warp -> team size), S (shared-memory slots), C (teams/SM cap).
Timing: one LSERK4 stage = one fused launch, CUDA events, mean of 5 steps after warm-up,
on an n x n A16 mesh (default n=362, K=262,088).  Oracle gate ("every timed variant
passes the oracle gate"): each variant also runs 100 steps of every (N, precision) on the jittered
12x12 mesh with the grid capped at 2 CTAs (each CTA walks 4-5 tiles: the full-size pipeline) and
is compared field by field with the fp64 oracle's fields stored in tests/golden/pipeline_gate_n12.npz
(tools/make_pipeline_gate_golden.py); `pick` disqualifies any variant whose per-field A14 error
exceeds 1e-12 (fp64) / 2e-5 (fp32).
"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, os.environ.get("TUNE_VDIR", "build_variants"))

GRID = {
    4: [dict(R=r, S=s, C=c, M=0) for r, s, c in itertools.product((6, 8, 11), (1, 2), (3, 5))],
    8: [dict(R=r, S=s, C=c, M=0) for r, s, c in itertools.product((4, 6, 8), (1, 2), (3, 5))]
    + [dict(R=8, S=s, C=c, M=1) for s, c in itertools.product((1, 2), (2, 3, 4, 6))],
}
if os.environ.get("TUNE_GRID") == "mma":  # only the fp64 tensor-core variants
    GRID = {8: [k for k in GRID[8] if k["M"] == 1]}
if os.environ.get("TUNE_GRID") == "tf2":  # fp32 3xTF32 with the field-split team (4 warps)
    GRID = {4: [dict(R=8, S=s, C=c, M=2, Q=q) for s, c, q in itertools.product((1, 2), (2, 3, 4, 6), (0, 1))]}
if os.environ.get("TUNE_GRID") == "all":  # every path: FMA, tensor-core (M=1), split teams (M=2)
    GRID = {4: [dict(R=r, S=s, C=c, M=0, Q=0) for r, s, c in itertools.product((6, 8, 11), (1, 2), (3, 5))]
            + [dict(R=8, S=s, C=c, M=1, Q=q) for s, c, q in itertools.product((1, 2), (3, 4, 6), (0, 1))]
            + [dict(R=8, S=s, C=c, M=2, Q=q) for s, c, q in itertools.product((1, 2), (2, 3, 4), (0, 1))]}
if os.environ.get("TUNE_GRID") == "m2":  # M=2 split teams (fp32 3xTF32 and fp64 DMMA), C>=1
    GRID = {4: [dict(R=8, S=s, C=c, M=2, Q=q) for s, c, q in itertools.product((1, 2), (1, 2, 3, 4), (0, 1))]}
if os.environ.get("TUNE_GRID") == "ff":  # flux-first phase order, every path, C up to 8
    GRID = {4: [dict(R=r, S=s, C=c, M=0, Q=0, F=1) for r, s, c in itertools.product((6, 8), (1, 2), (3, 5, 6))]
            + [dict(R=8, S=s, C=c, M=1, Q=q, F=1) for s, c, q in itertools.product((1, 2), (3, 4, 5, 6, 8), (0, 1))]
            + [dict(R=8, S=s, C=c, M=2, Q=1, F=1) for s, c in itertools.product((1, 2), (2, 3, 4))]}
if os.environ.get("TUNE_GRID") == "ff":  # + the current picks (volume first) for a same-box comparison
    _cur = json.load(open(os.path.join(ROOT, "paper_1304_5546_b200", "csrc", "tune.json")))
    GRID[0] = [dict(R=v["R"], S=v["S"], C=v["C"], M=v["M"], Q=v["Q"], F=0) for k, v in _cur.items()
               if not k.startswith("_")]
if os.environ.get("TUNE_GRID") == "og":  # tensor-core paths, flux first, operators via L1 (G=1)
    GRID = {4: [dict(R=8, S=s, C=c, M=m, Q=1, F=1, G=1) for s, c, m in itertools.product((1, 2), (4, 5, 6, 8), (1, 2))]
            + [dict(R=8, S=1, C=c, M=1, Q=1, F=f, G=0) for c, f in itertools.product((3, 4), (0, 1))]}
if os.environ.get("TUNE_GRID", "").startswith("file:"):  # a JSON list of variant names (a confirmation run)
    GRID = {0: [{x[0]: int(x[1:]) for x in v.split("_")} for v in json.load(open(os.environ["TUNE_GRID"][5:]))]}
if os.environ.get("TUNE_GRID") == "c5":  # fp64 N=8 (config C5): smaller teams (R=12/16) -> 2-3 CTAs/SM
    GRID = {8: [dict(R=r, S=s, C=c, M=0, F=f) for r, s, c, f in itertools.product((6, 8, 12, 16), (1, 2, 3),
                                                                               (1, 2, 3, 4), (0, 1))]
            + [dict(R=8, S=s, C=c, M=1, F=f) for s, c, f in itertools.product((1, 2, 3), (1, 2, 3), (0, 1))]}
if os.environ.get("TUNE_GRID") == "tf":  # tensor-core variants (fp32 3xTF32, fp64 DMMA)
    GRID = {4: [dict(R=8, S=s, C=c, M=1, Q=q) for s, c, q in itertools.product((1, 2), (3, 4, 6), (0, 1))]}


def name_of(k):
    return (f"R{k['R']}_S{k['S']}_C{k['C']}_M{k['M']}" + (f"_Q{k['Q']}" if "Q" in k else "")
            + (f"_F{k['F']}" if "F" in k else "") + (f"_G{k['G']}" if "G" in k else "")
            + (f"_X{k['X']}" if "X" in k else "") + (f"_I{k['I']}" if "I" in k else "")
            + (f"_W{k['W']}" if "W" in k else "")
            + "".join(f"_{x}{k[x]}" for x in ("Z", "U", "L", "Y") if x in k))


def cmd_build():
    from paper_1304_5546_b200 import build as B

    knobsets = {name_of(k): k for ks in GRID.values() for k in ks}
    for nm, k in sorted(knobsets.items()):
        lib = B.build_variant(nm, k, VDIR)
        import shutil
        shutil.rmtree(os.path.join(VDIR, nm), ignore_errors=True)  # keep only the .so (gpurun push size)
        print(lib, flush=True)


def cmd_measure(out):
    import numpy as np
    import torch

    import dginputs

    n = int(os.environ.get("TUNE_N", "362"))
    VX, VY, E = dginputs.rect_mesh(n)
    results = []
    libs = sorted(f for f in os.listdir(VDIR) if f.endswith(".so"))
    # each variant in a fresh process (one libdg.so per process)
    import subprocess

    for lib in libs:
        code = f"""
import sys, json; sys.path.insert(0, {ROOT!r})
import numpy as np, torch, dginputs
from paper_1304_5546_b200 import dg
VX, VY, E = dginputs.rect_mesh({n})
G = np.load({os.path.join(ROOT, "tests", "golden", "pipeline_gate_n12.npz")!r})
out = []
for N in range(1, 10):
    dt = dginputs.cfl_dt(VX, VY, E, N)
    for prec in (4, 8):
        try:
            c = dg.dg_setup(N, VX, VY, E, precision=prec)
        except dg.DGError as e:
            continue
        x, y = c.nodes()
        c.set_fields(*dginputs.cavity_mode(x, y, 0.0))
        c.run(dt, 3); c.sync()
        s = torch.cuda.ExternalStream(c.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); c.run(dt, 5); e1.record(s); e1.synchronize()
        ms = e0.elapsed_time(e1) / 25
        f = c.get_fields()
        c.destroy()
        # oracle gate: 100 steps on the stored case, grid capped (multi-tile pipeline), per-field A14
        g = c = dg.dg_setup(N, G["VX"], G["VY"], G["EToV"], precision=prec, max_ctas=2)
        xg, yg = g.nodes()
        q0 = dginputs.cavity_mode(xg, yg, float(G["t0_%d" % N]))
        q0 = tuple(a + b for a, b in zip(q0, dginputs.perturbation(xg.shape, float(G["amplitude"]), seed=N)))
        g.set_fields(*q0); g.run(float(G["dt%d" % N]), int(G["steps"])); got = g.get_fields(); g.destroy()
        gate = max(float(np.abs(a - G[nm + str(N)]).max() / np.abs(G[nm + str(N)]).max())
                   for a, nm in zip(got, ("Hx", "Hy", "Ez")))
        out.append(dict(N=N, prec=prec, ms=ms, chk=float(sum(np.abs(a).sum() for a in f)), gate=gate))
print(json.dumps(out))
"""
        env = dict(os.environ, DG_LIB=os.path.join(VDIR, lib))
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
        if p.returncode != 0:
            print(lib, "FAILED", p.stderr[-500:], flush=True)
            continue
        rows = json.loads(p.stdout.strip().splitlines()[-1])
        for r in rows:
            r["variant"] = lib[:-3]
        results += rows
        print(lib, " ".join(f"N{r['N']}p{r['prec']}:{r['ms']:.4f}" for r in rows), flush=True)
    with open(out, "w") as fh:
        json.dump(dict(n=n, results=results), fh, indent=1)


def cmd_pick(*paths):
    d = {"n": None, "results": []}
    for arg in paths:  # PATH or PATH:f32 / PATH:f64 (take only that precision's rows)
        path, _, only = arg.partition(":")
        dd = json.load(open(path))
        d["n"] = dd["n"]
        d["results"] += [r for r in dd["results"] if not only or only == ("f32" if r["prec"] == 4 else "f64")]
    path = "+".join(os.path.basename(x) for x in paths)  # noqa: keeps the :prec selectors
    best = {}
    chk = {}
    for r in d["results"]:
        key = f"N{r['N']}_{'f32' if r['prec'] == 4 else 'f64'}"
        tol = 1e-12 if r["prec"] == 8 else 2e-5
        if "gate" not in r or not r["gate"] <= tol:
            print("DISQUALIFIED (oracle gate)", key, r["variant"], r.get("gate", "not run"))
            continue
        chk.setdefault(key, r["chk"])
        if abs(r["chk"] - chk[key]) > 1e-6 * abs(chk[key]):
            print("WARNING: checksum mismatch", key, r["variant"])
            continue
        if key not in best or r["ms"] < best[key]["ms"]:
            best[key] = r
    tune = {"_doc": f"picked by tools/tune.py from {os.path.basename(path)} (fused stage, "
                    f"{d['n']}x{d['n']} A16 mesh): fastest knob set per (N, precision); M=1: tensor-core "
                    f"path (fp32 3xTF32 mma.sync, fp64 DMMA)"}
    for key, r in sorted(best.items()):
        k = dict(kv.split(":") for kv in [])
        parts = r["variant"].split("_")
        kn = {x[0]: int(x[1:]) for x in parts}
        kn.setdefault("M", 0)
        kn.setdefault("Q", 0)  # sweeps before the knob existed: register prefetch
        kn.setdefault("F", 0)  # sweeps before the knob existed: volume first
        kn.setdefault("G", 0)  # sweeps before the knob existed: operators in shared memory
        kn.setdefault("X", 0)  # sweeps before the knob existed: flux through shared memory
        kn.setdefault("I", 0)  # sweeps before the knob existed: products accumulator by accumulator
        kn.setdefault("W", 0)  # sweeps before the knob existed: streaming stores
        tune[key] = dict(kn, ms=round(r["ms"], 5))  # every knob letter of the variant name (Z, U, L, Y ...)
    out = os.path.join(ROOT, "paper_1304_5546_b200", "csrc", "tune.json")
    with open(out, "w") as fh:
        json.dump(tune, fh, indent=1)
    print(json.dumps(tune, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        cmd_build()
    elif sys.argv[1] == "measure":
        cmd_measure(sys.argv[2])
    elif sys.argv[1] == "pick":
        cmd_pick(*sys.argv[2:])
