mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gemm_tc_gpu.py -q -x -m gpu -k pool > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_iter.log
for rep in 1 2; do
  timeout 600 python tools/bench_ee.py 3 > gpurun_out/ab_rev.log 2>&1
  python - <<'PY'
import json, sys
for l in open('gpurun_out/ab_rev.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print('reversed pool', {k: round(d[k]['p50_batch_ms'], 4) for k in ('feedback_graph', 'feedback_graph_serial_ramps', 'vanilla_graph', 'compact_device_graph')})
PY
done
