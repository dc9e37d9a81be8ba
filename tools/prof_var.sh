# ncu (full set, source) of one fused stage launch per library variant:
#   bash tools/prof_var.sh TAG N PREC n MAT VARIANT...
#   (VARIANT main = the in-tree libdg.so, else build_modvar/TAG/VARIANT.so; MAT 1 = two-layer material)
TAG=$1; N=$2; PREC=$3; NN=$4; MAT=$5; shift 5
mkdir -p gpurun_out/pv
for v in "$@"; do
  if [ $v = main ]; then unset DG_LIB; else export DG_LIB=build_modvar/$TAG/$v.so; fi
  o=gpurun_out/pv/${TAG}_$v
  if [ "$MAT" = 1 ]; then prog="tools/prof_mat.py $N $PREC $NN 2"; else prog="tools/prof_one.py $N $PREC $NN 1 2"; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 7 -c 1 -o $o python $prog > $o.log 2>&1
  ncu -i $o.ncu-rep --page source --csv --print-source sass > ${o}_sass.csv 2>&1
  python tools/ncu_summary.py $o.ncu-rep > ${o}_summary.txt 2>&1
  rm -f $o.ncu-rep
done
