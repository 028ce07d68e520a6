# ncu launch lists of the vanilla and the EE feedback graphs (configs 1 and 3)
mkdir -p gpurun_out
for c in 1 3; do
  for r in vanilla ee; do
    timeout 600 ncu --nvtx --nvtx-include "$r/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_c${c}_$r.csv python tools/profile_ee_graph.py $c > /dev/null 2>&1; echo "ncu c$c $r rc=$?"
    python tools/launch_list_summary.py gpurun_out/ll_c${c}_$r.csv 25 > gpurun_out/ll_c${c}_$r.txt; head -12 gpurun_out/ll_c${c}_$r.txt
  done
done
timeout 900 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
