timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_distributed_gpu.py -q -x 2>&1 | tail -2
EEB200_TRACE_HOST=1 timeout 300 python tools/micro/e2e_trace.py 2>&1 | tail -12
timeout 300 python tools/micro/e2e_parts.py 2>&1 | tail -2
