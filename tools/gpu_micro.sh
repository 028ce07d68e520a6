#!/bin/bash
# Micro-benchmarks behind DESIGN.md's numbers, one file each under gpurun_out/.
mkdir -p gpurun_out
timeout 120 tools/micro/readbw > gpurun_out/micro_readbw.txt 2>&1
timeout 120 tools/micro/fold > gpurun_out/micro_fold.txt 2>&1
DIAG_VERSION=4 COPIES=1,4 MODES=eager,graph timeout 300 python tools/pipelined_sweeps.py > gpurun_out/micro_pipelined_sweeps.txt 2>&1
timeout 300 python tools/bench_axis.py > gpurun_out/micro_bench_axis.txt 2>&1
timeout 300 python tools/bench_ramp.py > gpurun_out/micro_bench_ramp.txt 2>&1
timeout 300 python tools/nccl_capture_check.py > gpurun_out/micro_nccl_capture.txt 2>&1
timeout 300 python tools/profile_tune.py > gpurun_out/micro_profile_tune.txt 2>&1
echo done
