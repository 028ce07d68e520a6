for r in 0 4 8; do
echo "reserve $r"
EEB200_RESERVE_PAIRS=$r timeout 900 python tools/bench_ee.py 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l)
    print({k: round(v['p50_batch_ms'],4) for k,v in d.items() if isinstance(v,dict) and 'p50_batch_ms' in v and 'graph' in k})
"
done
