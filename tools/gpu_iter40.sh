mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_convnet_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pt_iter.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_ll_c3_vanilla.csv python tools/profile_ee_graph.py 3 > /dev/null 2>&1; echo "ncu c3 rc=$?"
python tools/launch_list_summary.py gpurun_out/r02_ll_c3_vanilla.csv 30 > gpurun_out/r02_ll_c3_vanilla.txt; grep -i "maxpool\|total" gpurun_out/r02_ll_c3_vanilla.txt
