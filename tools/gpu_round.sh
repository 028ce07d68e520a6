#!/bin/bash
# One gpurun session: GPU parity tests, smoke, bench (+reference arm), EE + tune benches.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
timeout 600 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
timeout 300 python tools/bench_tune.py > gpurun_out/bench_tune.log 2>&1; echo "bench_tune rc=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-600
