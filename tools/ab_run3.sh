# A/B of the cluster instantiations on the bench (dev tool)
bench() { timeout 300 python bench.py --steps 4 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],2))"; }
bench auto
TTP_CK=lat bench lat
bench auto
