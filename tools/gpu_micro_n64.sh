mkdir -p gpurun_out
timeout 600 python tools/micro_gemm_n64.py > gpurun_out/micro_n64.jsonl 2>&1; echo "rc=$?"; cat gpurun_out/micro_n64.jsonl
