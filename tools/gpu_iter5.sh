mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_convnet_gpu.py -q -x > gpurun_out/pt_conv.log 2>&1; echo "pytest conv rc=$?"; tail -5 gpurun_out/pt_conv.log | cut -c1-300
timeout 600 python -m pytest tests/test_distributed_gpu.py -q -x > gpurun_out/pt_dist.log 2>&1; echo "pytest dist rc=$?"; tail -5 gpurun_out/pt_dist.log | cut -c1-300
c=3
timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_c${c}_vanilla_routed.csv python tools/profile_ee_graph.py $c > /dev/null 2>&1; echo "ncu c$c rc=$?"
python tools/launch_list_summary.py gpurun_out/ll_c${c}_vanilla_routed.csv 25 > gpurun_out/ll_c${c}_vanilla_routed.txt; head -8 gpurun_out/ll_c${c}_vanilla_routed.txt | cut -c1-150
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tune -s 2 -c 1 -o gpurun_out/prof_tune -f python tools/profile_tune.py > gpurun_out/ncu_tune.log 2>&1; echo "ncu tune rc=$?"
