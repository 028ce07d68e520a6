timeout 900 python -m pytest tests/test_ee_infer_gpu.py -k device_scheduled -q -x 2>&1 | tail -15
timeout 900 python tools/bench_ee.py 1 3 2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['config'])
    for k,v in d.items():
        if isinstance(v,dict) and 'samples_per_s' in v: print('  ',k, round(v['samples_per_s']), round(v.get('p50_batch_ms',0),4), v.get('matches_feedback_off_margin',''))
" 
