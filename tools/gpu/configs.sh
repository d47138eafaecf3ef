# every BASELINE config through bench.py (same contract line), one GPU
mkdir -p gpurun_out/configs
for c in ${CONFIGS:-1 2 3 5 4}; do
  extra=""
  [ "$c" = "5" ] && extra="--steps 3 --warmup 3"
  timeout 1500 python bench.py --config $c $extra > gpurun_out/configs/bench_cfg$c.json 2> gpurun_out/configs/bench_cfg$c.err
  echo "cfg$c rc=$?"; python -c "import json;d=json.load(open('gpurun_out/configs/bench_cfg$c.json'));print(d['config']['workload'], d['value'], d['e2e']['value'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'), d['parity']['ok'])" 2>&1 | tail -1
done
