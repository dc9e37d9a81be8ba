"""Summarise build/ptxas_<tag>.log: registers / spills / smem per stage-kernel instantiation."""
import glob, os, re, subprocess, sys
MODES = {0: "fused", 1: "volume", 2: "surf_rk", 3: "rhs", 4: "surface"}
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1304_5546_b200", "build")
pat = sys.argv[1] if len(sys.argv) > 1 else "*"
for log in sorted(glob.glob(os.path.join(root, f"ptxas_{pat}.log"))):
    tag = os.path.basename(log)[6:-4]
    txt = open(log).read()
    for m in re.finditer(r"Compiling entry function '(\S+)'.*?Used (\d+) registers", txt, re.S):
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        mm = re.search(r"stage_kernel<(\d), (\w+)>", name)
        if not mm:
            continue
        block = txt[m.start():m.end()]
        sp = re.findall(r"(\d+) bytes spill stores", block)
        print(f"{tag:8s} {MODES[int(mm.group(1))]:8s} mat={mm.group(2):5s} regs={m.group(2):>3s} spill={sp[-1] if sp else '?'}")
