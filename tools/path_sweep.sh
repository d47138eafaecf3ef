#!/bin/bash
# Throughput of each bond-kernel path per config (dev tool; prints one line per run).
for spec in "1 512" "3 512" "4 148" "4 296"; do
  set -- $spec
  for P in v0 cluster l2:1 l2:2 l2:4 l2:8; do
    out=$(TTP_BOND_PATH=$P timeout 300 python tools/run_cfg.py $1 $2 2 2>&1 | tail -1)
    echo "cfg$1 n=$2 $P $(echo "$out" | python -c 'import json,sys
try:
    d=json.loads(sys.stdin.read()); print(round(d["options_per_s"],1), round(d["kernels_ms"]["bond_kernel"],1))
except Exception as e: print("ERR", e)')"
  done
done
