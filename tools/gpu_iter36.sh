mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/micro_ln_pool.py > gpurun_out/micro_ln_pool.json 2>&1; echo "micro rc=$?"; cat gpurun_out/micro_ln_pool.json
timeout 900 python -m pytest tests/test_heads_gpu.py tests/test_gemm_tc_gpu.py tests/test_ee_parity_gpu.py tests/test_convnet_gpu.py tests/test_ee_infer_gpu.py tests/test_generative_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_iter.log
timeout 900 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/bench_ee.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print(d['config'], {k: round(d[k]['samples_per_s']) for k in d if isinstance(d[k], dict) and 'samples_per_s' in d[k]})
PY
