mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ee_infer_gpu.py tests/test_serve_live_gpu.py tests/test_heads_gpu.py -q -x 2>&1 | tail -3
for c in 1 3; do
timeout 900 python tools/bench_ee.py $c 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['config'])
    for k,v in d.items():
        if isinstance(v,dict) and 'samples_per_s' in v: print('  ',k, round(v['samples_per_s']), round(v.get('p50_batch_ms',0),4))
"
done
timeout 600 ncu --nvtx --nvtx-include "ee/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_c1_ee.csv python tools/profile_ee_graph.py 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_list_summary.py gpurun_out/ll_c1_ee.csv 20 | cut -c1-150
