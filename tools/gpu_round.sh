#!/bin/bash
# One gpurun session: GPU parity tests, smoke, bench (+reference arm), the EE and
# tune benches on their own, and the ncu launch lists of the EE graphs.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest ${PYTEST_SEL:-tests} -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log | cut -c1-400
