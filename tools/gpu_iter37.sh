mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/micro_ln_pool.py > gpurun_out/micro_ln_pool.json 2>&1; echo "micro rc=$?"; cut -c1-400 gpurun_out/micro_ln_pool.json
timeout 900 python -m pytest tests/test_generative_gpu.py tests/test_ee_parity_gpu.py tests/test_ee_infer_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_iter.log
