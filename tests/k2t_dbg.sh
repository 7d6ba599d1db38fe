#!/bin/bash
# K2t debug-switch sweep on one cell (GPU box): SI_K2_DEBUG bits of spmm_tcx.cu
cell=${1:-c5b}
for d in 0 1 8192 9 512 16 48 57 569; do
  echo -n "debug=$d  "; SI_K2_DEBUG=$d timeout 120 python tests/prof_one.py $cell tc 10 nk 2>&1 | tail -1
done
