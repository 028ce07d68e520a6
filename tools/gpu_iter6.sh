mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_ordered_sum_gpu.py -q -x > gpurun_out/pt_osum.log 2>&1; echo "pytest osum rc=$?"; tail -15 gpurun_out/pt_osum.log | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tune or grid" > gpurun_out/pt_tune.log 2>&1; echo "pytest tune rc=$?"; tail -5 gpurun_out/pt_tune.log | cut -c1-300
timeout 600 python tools/bench_tune.py > gpurun_out/bench_tune.log 2>&1; echo "bench_tune rc=$?"; tail -1 gpurun_out/bench_tune.log | cut -c1-700
timeout 600 python tools/bench_gen.py > gpurun_out/bench_gen.log 2>&1; echo "bench_gen rc=$?"; tail -1 gpurun_out/bench_gen.log | cut -c1-900
