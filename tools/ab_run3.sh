# A/B of library variants on the bench (dev tool): base vs tools/alt/lib_*.so
bench() { timeout 300 python bench.py --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],2))"; }
cp paper_2203_02804_b200/libttpricer_b200.so /tmp/base.so
bench base
for v in "$@"; do
  cp tools/alt/lib_$v.so paper_2203_02804_b200/libttpricer_b200.so
  bench $v
done
cp /tmp/base.so paper_2203_02804_b200/libttpricer_b200.so
bench base
