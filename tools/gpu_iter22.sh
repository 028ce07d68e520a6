mkdir -p gpurun_out
timeout 300 python tools/osum_diag.py 2>&1 | tail -6
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tune -s 1 -c 1 -o gpurun_out/tune_full -f python tools/tune_phases.py > gpurun_out/ncu_tune.log 2>&1; echo "ncu rc=$?"
