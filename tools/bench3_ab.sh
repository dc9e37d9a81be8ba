# Same-box A/B of the 3D order sweep: the in-tree library against a variant library (here the
# PF=0 build of the surface-prefetch experiment, packed as build_modvar/v3/pf0.so by hand; see
# profiles/r02_bench3d_pf_ab.txt).  Run on the GPU box from the repo root.
tar xzf build_modvar.tgz
for lib in main build_modvar/v3/pf0.so; do
 for prec in 4 8; do for n in 1 2 3 4 5; do
  if [ $lib = main ]; then unset DG_LIB; else export DG_LIB=$lib; fi
  python bench.py --dim 3 --order $n --prec $prec --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', $prec, $n, '%.4g'%d['value'], d['ms_per_step'])"
 done; done
done
