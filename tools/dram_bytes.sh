#!/bin/bash
# DRAM bytes and duration per fused stage launch (ncu, 5 launches = one LSERK4 step) of the default
# library and the connectivity-compression builds (build_variants/allz1.so: connectivity words,
# allz2.so: geometry only) for N = 2 and N = 5 (C4), fp32 and fp64.  Output: gpurun_out/dram_<lib>_N<n>_p<p>.csv
mkdir -p gpurun_out
for L in main allz1 allz2; do
  if [ $L = main ]; then export DG_LIB=""; else export DG_LIB=build_variants/$L.so; fi
  for N in 2 5; do for P in 4 8; do
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        -k regex:stage_kernel -s 10 -c 5 --csv --log-file gpurun_out/dram_${L}_N${N}_p${P}.csv \
        python tools/prof_one.py $N $P 724 1 3 > /dev/null 2>&1
  done; done
done
python - <<'PY'
import csv, glob, collections
rows = collections.defaultdict(dict)
for f in sorted(glob.glob("gpurun_out/dram_*_N*_p*.csv")):
    tag = f.split("dram_")[1][:-4]
    lib, n, p = tag.split("_")
    vals = collections.defaultdict(list)
    for r in csv.DictReader(l for l in open(f) if l.startswith('"')):
        try:
            vals[r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
        except (KeyError, ValueError):
            pass
    if vals:
        b = (sum(vals["dram__bytes_read.sum"]) + sum(vals["dram__bytes_write.sum"])) / len(vals["dram__bytes_read.sum"])
        t = sum(vals["gpu__time_duration.sum"]) / len(vals["gpu__time_duration.sum"])
        rows[(n, p)][lib] = (b, t)
for (n, p), d in sorted(rows.items()):
    base = d.get("main")
    print(n, p, "  ".join(f"{lib}: {b/1e6:8.1f} MB {t:8.1f} {'' if not base else f'({b/base[0]-1:+.1%} bytes, {t/base[1]-1:+.1%} time)'}"
                           for lib, (b, t) in sorted(d.items())))
PY
