timeout 900 python tools/profile_compact.py 3 2>&1 | tail -1
timeout 900 python tools/profile_compact.py 1 2>&1 | tail -1
