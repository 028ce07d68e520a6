mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_heads_gpu.py tests/test_ee_infer_gpu.py tests/test_ee_parity_gpu.py tests/test_serve_live_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_iter.log
timeout 600 python tools/bench_ee.py 1 > gpurun_out/bench_ee1.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/bench_ee1.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print({k: (round(d[k]['samples_per_s']), round(d[k]['p50_batch_ms'], 4)) for k in d if isinstance(d[k], dict) and 'samples_per_s' in d[k]})
PY
timeout 600 python tools/bench_ramp.py > gpurun_out/r02_micro_bench_ramp.txt 2>&1; echo "ramp rc=$?"; tail -2 gpurun_out/r02_micro_bench_ramp.txt
