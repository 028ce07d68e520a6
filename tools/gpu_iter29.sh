timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_serve_live_gpu.py -k "tune or closed_loop" -q -x 2>&1 | tail -2
timeout 300 python tools/tune_phases.py 2>&1 | tail -2
timeout 600 python tools/bench_tune.py 2>&1 | tail -1 | cut -c1-520
