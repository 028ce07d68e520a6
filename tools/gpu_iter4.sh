mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_convnet_gpu.py tests/test_gemm_tc_gpu.py -q -x > gpurun_out/pt_conv.log 2>&1; echo "pytest conv rc=$?"; tail -25 gpurun_out/pt_conv.log | cut -c1-300
timeout 900 python -m pytest tests/test_ee_infer_gpu.py tests/test_ee_parity_gpu.py -q -x > gpurun_out/pt_ee.log 2>&1; echo "pytest ee rc=$?"; tail -15 gpurun_out/pt_ee.log | cut -c1-300
for c in 3 1; do
  timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_c${c}_vanilla_routed.csv python tools/profile_ee_graph.py $c > /dev/null 2>&1; echo "ncu c$c rc=$?"
  python tools/launch_list_summary.py gpurun_out/ll_c${c}_vanilla_routed.csv 25 > gpurun_out/ll_c${c}_vanilla_routed.txt; head -14 gpurun_out/ll_c${c}_vanilla_routed.txt | cut -c1-150
done
timeout 900 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/bench_ee.log'):
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['config'])
    for k,v in d.items():
        if isinstance(v,dict): print('  ',k, {a:(round(b,4) if isinstance(b,float) else b) for a,b in v.items()})
PY
