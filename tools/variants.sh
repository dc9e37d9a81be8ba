#!/bin/bash
# time C4 (fp32 / fp64 fused) for each libdg variant in build_variants/*.so
for so in build_variants/*.so; do
  echo "== $so"
  DG_LIB=$PWD/$so python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
from probe import probe
probe(5, 4, 724, True); probe(5, 8, 724, True)
" 2>&1 | grep -v Warn
done
