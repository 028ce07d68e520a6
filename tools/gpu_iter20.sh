mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ordered_sum_gpu.py tests/test_gpu_parity.py -k "ordered or sequential or many_rows or tune" -q -x 2>&1 | tail -4
timeout 300 python tools/tune_phases.py 2>&1 | tail -3
timeout 600 python tools/bench_tune.py 2>&1 | tail -1 | cut -c1-600
