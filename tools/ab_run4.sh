# A/B: base, library variants and env knobs, interleaved twice (dev tool)
bench() { timeout 300 env $2 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],2))"; }
cp paper_2203_02804_b200/libttpricer_b200.so /tmp/base.so
for rep in 1 2; do
  cp /tmp/base.so paper_2203_02804_b200/libttpricer_b200.so
  bench base X=1
  [ -n "$LAZY2" ] && bench lazy2 TTP_LAZY=2
  for v in "$@"; do
    cp tools/alt/lib_$v.so paper_2203_02804_b200/libttpricer_b200.so
    bench $v X=1
  done
done
cp /tmp/base.so paper_2203_02804_b200/libttpricer_b200.so
