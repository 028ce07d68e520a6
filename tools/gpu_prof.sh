#!/bin/bash
# ncu only: launch list + full capture of the sweep kernels for family $1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python tools/profile_sweep.py ${1:-diagonal} 20 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_diag2|k_keys|k_count' -s 3 -c 2 -o gpurun_out/prof_sweep -f python tools/profile_sweep.py ${1:-diagonal} 8 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
