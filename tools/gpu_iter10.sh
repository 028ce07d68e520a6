mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_generative_gpu.py -q -x > gpurun_out/pt_gen.log 2>&1; echo "pytest gen rc=$?"; tail -25 gpurun_out/pt_gen.log | cut -c1-300
timeout 600 python tools/bench_gen.py > gpurun_out/bench_gen.log 2>&1; echo "bench_gen rc=$?"; tail -2 gpurun_out/bench_gen.log | cut -c1-1200
