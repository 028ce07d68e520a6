mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_convnet_gpu.py tests/test_gemm_tc_gpu.py -q -x 2>&1 | tail -2
timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_c3_v.csv python tools/profile_ee_graph.py 3 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_list_summary.py gpurun_out/ll_c3_v.csv 8 | cut -c1-150
