# usage: bash ab.sh tag   (run on the GPU box)
TAG=$1
TTP_SWAP_FILTER=1 timeout 300 python tools/phase_timing.py 2>&1 | grep -A2 "cfg4 batch 148" > gpurun_out/pt_$TAG.log
for v in 1 0 1 0; do TTP_SWAP_FILTER=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_${TAG}_$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab_${TAG}_$v.json'));print('filter=$v', round(d['value'],1))" >> gpurun_out/ab_$TAG.log; done
