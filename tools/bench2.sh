# two bench runs, printing value / e2e / per-kernel launch ms (dev tool)
for i in 1 2; do
timeout 300 python bench.py --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],2), [(x['kernel'], round(x['avg_launch_ms'],2), round(x['frac'],3)) for x in d['roofline_secondary']])"
done
