# A/B of the diagonal sweep versions (4: last-CTA finalise, 6: scan-merge-ticket)
# plus the cluster-split ramp heads.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
EEB200_DIAG_VERSION=6 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_heads_gpu.py -q -x > gpurun_out/pt_diag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_diag.log
OWNFLUSH=1 timeout 300 python tools/ab_diag.py 4 6 4 6 > gpurun_out/ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab.log | tail -4
timeout 300 python tools/trace_diag.py 4 6 > gpurun_out/trace.log 2>&1; echo "trace rc=$?"; cat gpurun_out/trace.log | tail -4
for v in 4 6; do DIAG_VERSION=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_v$v.csv python tools/profile_sweep.py diagonal 30 > /dev/null 2>&1; echo "ncu $v rc=$?"; done
timeout 300 python tools/bench_ramp.py > gpurun_out/bench_ramp.log 2>&1; echo "ramp rc=$?"; cat gpurun_out/bench_ramp.log | tail -2
for v in 4 6; do EEB200_DIAG_VERSION=$v timeout 600 python bench.py > gpurun_out/bench_v$v.log 2>&1; echo "bench $v rc=$?"; tail -1 gpurun_out/bench_v$v.log | cut -c1-200; done
timeout 600 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
