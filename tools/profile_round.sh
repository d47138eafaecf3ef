#!/bin/bash
# Round profile: launch list of one bench run, then one full ncu capture per
# top kernel (each capture only after the plain command exited 0).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_plain.json 2> $OUT/bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_list.log 2>&1
for K in cluster_bond_kernel conv_site_dmma tt_inner; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/$K \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_$K.log 2>&1
done
