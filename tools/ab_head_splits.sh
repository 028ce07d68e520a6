mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for rep in 1 2; do for s in 0 2 1; do
  EEB200_HEAD_SPLITS=$s timeout 600 python tools/bench_ee.py 3 > gpurun_out/ab_h$s.log 2>&1
  python - $s <<'PY'
import json, sys
for l in open(f'gpurun_out/ab_h{sys.argv[1]}.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print('splits=' + sys.argv[1], {k: round(d[k]['p50_batch_ms'], 4) for k in ('feedback_graph', 'feedback_graph_serial_ramps', 'vanilla_graph', 'compact_device_graph')})
PY
done; done
