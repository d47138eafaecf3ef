#!/bin/bash
# A/B of library variants (gpurun_variants_<name>.so at the repo root, built
# by hand from csrc/build/*.o with one object swapped) against the in-tree
# release library: bench lines per config, interleaved repetitions.
# Usage: VARIANTS="default t0" CFGS="4 1" REPS=2 tools/ab_lib_variants.sh
OUT=gpurun_out/ab_variants
mkdir -p $OUT
LIB=paper_2203_02804_b200/libttpricer_b200.so
cp $LIB /tmp/lib_default.so
for rep in $(seq 1 ${REPS:-2}); do
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then cp /tmp/lib_default.so $LIB; else cp gpurun_variants_$v.so $LIB; fi
  for c in ${CFGS:-4}; do
    python bench.py --config $c --steps ${STEPS:-4} --warmup 3 --no-cpu-baseline > $OUT/${v}_cfg${c}_$rep.json 2> $OUT/${v}_cfg${c}_$rep.err
    python -c "
import json,sys
d=json.loads(open('$OUT/${v}_cfg${c}_$rep.json').read().strip().splitlines()[-1])
print('$v cfg$c', round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],1), d['parity']['ok'], round(d['parity']['max_band_ratio'],2), {k:(v['launches'],round(v['ms'],1)) for k,v in d['kernels'].items() if 'bond' in k}, flush=True)
" 2>&1 | tail -1
  done
done
done
cp /tmp/lib_default.so $LIB
