timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
EEB200_TRACE_HOST=1 timeout 300 python tools/micro/e2e_trace.py 2>&1 | tail -6
timeout 300 python tools/micro/e2e_parts.py 2>&1 | tail -2
