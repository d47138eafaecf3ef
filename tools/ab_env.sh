# A/B of env knobs on the bench, interleaved (dev tool): ab_env.sh "NAME=VAL" ...
bench() { timeout 300 env $2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],2))"; }
for rep in 1 2; do
  bench default X=1
  for kv in "$@"; do bench "$kv" "$kv"; done
done
