mkdir -p gpurun_out
c=3
timeout 600 python -m pytest tests/test_convnet_gpu.py -q -x 2>&1 | tail -2; timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_c${c}_vanilla_routed.csv python tools/profile_ee_graph.py $c > /dev/null 2>&1; echo "ncu c$c rc=$?"
python tools/launch_list_summary.py gpurun_out/ll_c${c}_vanilla_routed.csv 25 > gpurun_out/ll_c${c}_vanilla_routed.txt; head -12 gpurun_out/ll_c${c}_vanilla_routed.txt | cut -c1-150
