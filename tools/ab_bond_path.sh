#!/bin/bash
# A/B of the bond kernel path for one config through the dev library's
# TTP_BOND_PATH knob (auto | l2:C global-slice clusters | cluster = shared-
# memory clusters | v0 = one CTA per instance).
# Usage: CFG=3 PATHS="auto l2:1 l2:2 cluster" tools/ab_bond_path.sh
set -u
CFG=${CFG:-3}
OUT=gpurun_out/ab_path_cfg$CFG
mkdir -p $OUT
for rep in 1 2; do
for p in ${PATHS:-auto l2:1 l2:2 cluster}; do
  tag=${p//:/_}
  if [ "$p" = auto ]; then unset TTP_BOND_PATH; else export TTP_BOND_PATH=$p; fi
  TTP_DEV_LIBRARY=1 timeout 600 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > $OUT/${tag}_$rep.json 2> $OUT/${tag}_$rep.err
  python - $OUT/${tag}_$rep.json "$p" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "ms", round(d["ms_per_step"], 1),
          "parity", d["parity"]["ok"], round(d["parity"]["max_band_ratio"], 2),
          {k: (v["launches"], round(v["ms"], 1)) for k, v in d["kernels"].items() if "bond" in k}, flush=True)
except Exception as e:
    print(sys.argv[2], "FAILED", e, flush=True)
PY
done
done
