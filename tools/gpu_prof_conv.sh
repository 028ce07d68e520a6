mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_pair -s 2 -c 1 -o gpurun_out/conv3x3 -f python tools/profile_conv.py 3x3 > gpurun_out/ncu_conv.log 2>&1; echo "ncu 3x3 rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_pair -s 2 -c 1 -o gpurun_out/conv1x1 -f python tools/profile_conv.py 1x1 >> gpurun_out/ncu_conv.log 2>&1; echo "ncu 1x1 rc=$?"
