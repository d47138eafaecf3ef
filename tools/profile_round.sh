#!/bin/bash
# Round profile of one bench config (default 4): the plain run, then the ncu
# launch list of the same command, then one full capture per top kernel --
# each ncu pass only after the plain command exited 0.  Summarise here with
#   python tools/ncu_summary.py gpurun_out/prof_cfg$CFG r02 --config=$CFG
set -u
CFG=${CFG:-4}
OUT=gpurun_out/prof_cfg$CFG
mkdir -p $OUT
python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_plain.json 2> $OUT/bench_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_list.log 2>&1
for K in ${KERNELS:-cluster_bond_kernel conv_site_dmma tt_inner}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 -o $OUT/$K \
      python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_$K.log 2>&1
done
