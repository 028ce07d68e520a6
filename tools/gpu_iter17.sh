mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_convnet_gpu.py -q -x 2>&1 | tail -3
timeout 600 python -m pytest tests/test_ee_infer_gpu.py -q -x 2>&1 | tail -2
timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_c1_v.csv python tools/profile_ee_graph.py 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_list_summary.py gpurun_out/ll_c1_v.csv 8 | cut -c1-150
timeout 900 python tools/bench_ee.py 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['config'])
    for k,v in d.items():
        if isinstance(v,dict): print('  ',k, {a:(round(b,4) if isinstance(b,float) else b) for a,b in v.items()})
"
