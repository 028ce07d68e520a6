mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_serve_live_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_iter.log
timeout 600 python tools/bench_serve_live.py > gpurun_out/serve_live.log 2>&1; echo "serve rc=$?"; tail -1 gpurun_out/serve_live.log
