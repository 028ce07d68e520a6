timeout 300 python tools/osum_diag.py 2>&1 | tail -6
timeout 600 python -m pytest tests/test_ordered_sum_gpu.py tests/test_gpu_parity.py -k "ordered or sequential or many_rows or tune" -q -x 2>&1 | tail -2
timeout 300 python tools/tune_phases.py 2>&1 | tail -3
