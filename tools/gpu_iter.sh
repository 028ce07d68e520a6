# iteration check: EE pipeline tests (compaction runner, overlapped ramps, heads),
# the sweep A/B, ramp micro-bench, EE bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_ee_infer_gpu.py tests/test_heads_gpu.py tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_iter.log
OWNFLUSH=1 timeout 300 python tools/ab_diag.py 4 6 4 6 > gpurun_out/ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab.log | tail -4
for v in 4 6; do EEB200_DIAG_VERSION=$v timeout 600 python bench.py --steps 300 > gpurun_out/bench_v$v.log 2>&1; echo "bench $v rc=$?"; tail -1 gpurun_out/bench_v$v.log | cut -c1-200; done
timeout 900 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
