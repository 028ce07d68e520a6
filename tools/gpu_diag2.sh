#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "diag or full_size or medium or golden" > gpurun_out/pytest_diag.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_diag.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], json.dumps(d['roofline']))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python tools/profile_sweep.py diagonal 20 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_diag' -s 3 -c 1 -o gpurun_out/prof_diag -f python tools/profile_sweep.py diagonal 8 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
