#!/bin/bash
# A/B of two library builds on the Random-dense regimes (pair kernel time per variant)
for lib in "$@"; do
  for d in 0.01 0.03 0.09; do
    TDS_LIB=paper_1410_2698_b200/$lib python tools/prof_dense.py $d 50880 temporal 2>&1 | tail -1 | sed "s/^/$lib d=$d T /"
  done
  TDS_LIB=paper_1410_2698_b200/$lib python tools/prof_dense.py 0.03 50880 spatiotemporal 2>&1 | tail -1 | sed "s/^/$lib d=0.03 ST /"
done
