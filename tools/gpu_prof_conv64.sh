mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_pair -s 2 -c 1 -o gpurun_out/conv1x1_64 -f python tools/profile_conv.py 1x1_64 > gpurun_out/ncu_conv64.log 2>&1; echo "ncu rc=$?"
