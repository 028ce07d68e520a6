mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_tune -s 26 -c 1 -o gpurun_out/prof_tune1000 -f python tools/profile_tune.py > gpurun_out/ncu_tune.log 2>&1; echo "ncu tune rc=$?"
