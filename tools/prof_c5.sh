# ncu (full set, source) of one fused N=8 fp64 material stage launch per library variant:
#   bash tools/prof_c5.sh VARIANT...   (main = the in-tree libdg.so; else build_modvar/N8_f64/VARIANT.so)
mkdir -p gpurun_out/p5
for v in "$@"; do
  if [ $v = main ]; then unset DG_LIB; else export DG_LIB=build_modvar/N8_f64/$v.so; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 7 -c 1 -o gpurun_out/p5/$v python tools/prof_mat.py 8 8 512 2 > gpurun_out/p5/$v.log 2>&1
  ncu -i gpurun_out/p5/$v.ncu-rep --page source --csv --print-source sass > gpurun_out/p5/${v}_sass.csv 2>&1
  ncu -i gpurun_out/p5/$v.ncu-rep --page raw --csv > gpurun_out/p5/${v}_raw.csv 2>&1
  python tools/ncu_summary.py gpurun_out/p5/$v.ncu-rep > gpurun_out/p5/${v}_summary.txt 2>&1
done
rm -f gpurun_out/p5/*.ncu-rep
