mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_diag3_windows_db -s 1 -c 1 -o gpurun_out/r02_k_diag3_windows_db -f python tools/profile_windows.py 20 > gpurun_out/r02_ncu_w.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 50 --warmup 3 --no-extra --no-cpu-baseline --no-replicas > gpurun_out/r02_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
