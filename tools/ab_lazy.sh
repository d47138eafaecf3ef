# A/B of the deferred-update flush cadence (TTP_LAZY) with filtered swap passes (GPU box)
TAG=$1; shift
for rep in 1 2; do for f in "$@"; do TTP_LAZY=$f timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lz_${TAG}_$f.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/lz_${TAG}_$f.json'));print('lazy=$f', round(d['value'],1))" >> gpurun_out/lz_$TAG.log; done; done
