#!/bin/bash
# ncu --set full of the secondary kernels (dense sum, fiber evaluators, Monte
# Carlo), each only after its plain command exited 0.
set -u
OUT=gpurun_out/prof2
mkdir -p $OUT
cap() {  # cap <mode> <ncu -k filter> <name>
  python tools/kernel_rooflines.py $1 > $OUT/plain_$3.log 2>&1 || { echo "plain $1 failed"; return; }
  ncu --set full --clock-control none --import-source on -k $2 -c 1 -o $OUT/$3 \
      python tools/kernel_rooflines.py $1 > $OUT/ncu_$3.log 2>&1
  tail -1 $OUT/ncu_$3.log
}
cap dense regex:dense_partial dense_partial_kernel
cap fiber "regex:fiber_fast -s 4" fiber_fast_kernel
cap fiber bond_kernel bond_kernel_v0
cap mc regex:mc_path mc_path_kernel
cap inner64 regex:tt_inner_split tt_inner_split_kernel
