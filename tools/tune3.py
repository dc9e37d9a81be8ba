"""Knob sweep of the 3D kernels (the paper's "looping over all variants and
comparing timing data").

    python tools/tune3.py build     # CPU: one library per knob set -> build_variants3/
    python tools/tune3.py run       # GPU: bench.py --dim 3 for every (variant, N, precision) -> JSONL
    python tools/tune3.py pick FILE # print the per-(N, precision) best knobs as tune.json entries

Knobs (build.py inst_source3): RS surface rows per warp, SQ surface kernel stages the tile's fields
by TMA.  Every variant is checked for parity by tests/test_gpu_3d.py only once picked into tune.json.
"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build_variants3")
GRID = [dict(SQ=sq, RS=rs) for sq, rs in itertools.product((0, 1), (2, 4, 8))]
# second pass (after the first picked RS = 2 almost everywhere): RS = 1, and the volume kernel's R
GRID2 = [dict(SQ=sq, RS=1) for sq in (0, 1)] + [dict(SQ=sq, RS=2, R=r) for sq, r in itertools.product((0, 1), (4, 16))]
# third pass: RS = 1 (N <= 3 picks) and RS = 4 (N = 4 fp32 pick) with the volume R
GRID3 = [dict(SQ=sq, RS=1, R=r) for sq, r in itertools.product((0, 1), (4, 16))] + [dict(SQ=1, RS=4, R=r) for r in (4, 16)]
# fused-stage pass (round 2): the fused kernel's rows per warp RF (its other knobs are RF-only)
GRIDF = [dict(RF=r) for r in (1, 2, 4, 8)]
# the fused kernel's volume by derivative sums (VS = 1) against the W form (VS = 0)
GRIDV = [dict(VS=v, RF=r) for v in (0, 1) for r in (1, 2, 4)]
# resident fused CTAs per SM the registers are sized for (F3C), on top of each module's tuned RF / VS
GRIDC = [dict(F3C=c) for c in (2, 3, 4)]
GRIDD = [dict(D3=1)]  # double-buffered fused tiles (A/B against main)
GRIDR = [dict(RF=r, G3=g) for r in (1, 2, 4) for g in (0, 2)]  # RF re-tune with the code preload
GRIDG = [dict(G3=2), dict(G3=1)]  # neighbour codes preloaded (2), + cp.async gathers (1), A/B against main (0)
GRID = {"2": GRID2, "3": GRID3, "fused": GRIDF, "vs": GRIDV, "f3c": GRIDC, "g3": GRIDG, "d3": GRIDD, "rfg": GRIDR}.get(os.environ.get("TUNE3_GRID", ""), GRID)


def name(k):
    return "_".join(f"{a}{b}" for a, b in sorted(k.items()))


def build():
    from paper_1304_5546_b200 import build as B

    for k in GRID:
        print(B.build_variant3(name(k), k, VDIR, merge=os.environ.get("TUNE3_GRID") in ("f3c", "g3", "d3", "rfg")), flush=True)


def run(out="gpurun_out/tune3.jsonl", steps=20):
    for k in GRID:
        lib = os.path.join(VDIR, name(k) + ".so")
        for prec, n in itertools.product((4, 8), range(1, 6)):
            cmd = [sys.executable, "bench.py", "--dim", "3", "--order", str(n), "--prec", str(prec), "--steps",
                   str(steps), "--warmup", "3", "--no-cpu-baseline"]
            r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, DG_LIB=lib), capture_output=True, text=True,
                               timeout=300)
            lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
            rec = dict(knobs=k, N=n, prec=prec, rc=r.returncode)
            if lines:
                d = json.loads(lines[-1])
                rec.update(value=d.get("value"), ms_per_step=d.get("ms_per_step"))
            else:
                rec["err"] = r.stderr[-400:]
            print(json.dumps(rec), flush=True)
            with open(os.path.join(ROOT, out), "a") as fh:
                fh.write(json.dumps(rec) + "\n")


def pick(path):
    best = {}
    for l in open(path):
        d = json.loads(l)
        if d.get("value") is None:
            continue
        key = f"3d_N{d['N']}_f{32 if d['prec'] == 4 else 64}"
        if key not in best or d["value"] > best[key]["value"]:
            best[key] = d
    for key, d in sorted(best.items()):
        print(f'"{key}": {json.dumps(d["knobs"])},  # {d["value"]:.4g} DOF/s')


if __name__ == "__main__":
    {"build": build, "run": run, "pick": lambda: pick(sys.argv[2])}[sys.argv[1]]()
