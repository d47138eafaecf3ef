cp paper_2203_02804_b200/libttpricer_b200.so /tmp/base.so
for v in base ic256 ic256sc2; do
  if [ $v = base ]; then cp /tmp/base.so paper_2203_02804_b200/libttpricer_b200.so; else cp tools/alt/lib_$v.so paper_2203_02804_b200/libttpricer_b200.so; fi
  python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "p1 or inner" 2>&1 | tail -1
  timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['e2e']['value'],1), [(x['kernel'], round(x['avg_launch_ms'],2)) for x in d['roofline_secondary']])"
done
cp /tmp/base.so paper_2203_02804_b200/libttpricer_b200.so
