mkdir -p gpurun_out
timeout 300 python tools/tune_phases.py 2>&1 | tail -3
timeout 600 python tools/bench_tune.py 2>&1 | tail -1 | cut -c1-700
