mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for s in 8 4 2 1; do
  EEB200_EXIT_MAX_S=$s timeout 600 python tools/bench_ee.py 1 > gpurun_out/bench_ee_s$s.log 2>&1
  python - $s <<'PY'
import json, sys
for l in open(f'gpurun_out/bench_ee_s{sys.argv[1]}.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print('S<=' + sys.argv[1], {k: (round(d[k]['samples_per_s']), round(d[k]['p50_batch_ms'], 4)) for k in ('feedback_graph', 'feedback_graph_serial_ramps', 'vanilla_graph', 'compact_device_graph')})
PY
done
