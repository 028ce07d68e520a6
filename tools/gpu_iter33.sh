# iteration: GELU epilogue + graph-replayed serving loop
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_serve_live_gpu.py tests/test_gemm_tc_gpu.py tests/test_ee_parity_gpu.py tests/test_ee_infer_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt_iter.log
timeout 600 python tools/bench_gemm3.py > gpurun_out/gemm3.jsonl 2>&1; echo "gemm3 rc=$?"; grep -E '"bert_fc1"|"bert_qkv"' gpurun_out/gemm3.jsonl | cut -c1-240
timeout 600 python tools/bench_serve_live.py > gpurun_out/serve_live.log 2>&1; echo "serve rc=$?"; tail -1 gpurun_out/serve_live.log
