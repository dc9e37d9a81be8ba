"""Write profiles/traffic.json: DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
of the fused stage kernel, mean over the launches in an `ncu --set full` capture of one LSERK4 step
(5 launches = 5 stages).  bench.py reads it for roofline.traffic.

    python tools/traffic.py KEY=REPORT.ncu-rep [KEY=REPORT.ncu-rep ...]
    (KEY = N<order>_p<bytes>_n<cells>_P<ranks>_<kernel>, e.g. N5_p4_n724_P1_fused)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        b = sum(float(d[k]) * SCALE[units[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res.append((d.get("Kernel Name", ""), b))
    return res


def main():
    out = os.environ.get("TRAFFIC_OUT", os.path.join(ROOT, "profiles", "traffic.json"))
    tab = json.load(open(out)) if os.path.exists(out) else {}
    tab["_doc"] = ("DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the fused "
                   "stage kernel, ncu --set full, mean over the 5 launches (LSERK4 stages) of one step "
                   "(tools/traffic.py).  Keys: N<order>_p<bytes>_n<cells>_P<ranks>_<kernel>.  Read by "
                   "bench.py for roofline.traffic.")
    for arg in sys.argv[1:]:
        key, path = arg.split("=", 1)
        ls = launches(path)
        if key.endswith("_split"):  # a split-variant capture: volume = stage_kernel<1, .>, surface = <2, .>
            groups = {key[:-6] + "_volume": [b for n, b in ls if "stage_kernel<1" in n.replace("(int)", "")],
                      key[:-6] + "_surface": [b for n, b in ls if "stage_kernel<2" in n.replace("(int)", "")]}
        else:
            groups = {key: [b for _, b in ls]}
        for k, b in groups.items():
            tab[k] = sum(b) / len(b)
            print(k, len(b), "launches", [f"{x / 1e9:.3f}" for x in b], f"mean {tab[k] / 1e9:.4f} GB")
    with open(out, "w") as fh:
        json.dump(tab, fh, indent=1)


if __name__ == "__main__":
    main()
