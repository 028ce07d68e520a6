mkdir -p gpurun_out
for r in vanilla ee; do
timeout 600 ncu --nvtx --nvtx-include "$r/" --graph-profiling node --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_c5_$r.csv python tools/profile_gen.py > /dev/null 2>&1; echo "ncu $r rc=$?"
python tools/launch_list_summary.py gpurun_out/ll_c5_$r.csv 16 > gpurun_out/ll_c5_$r.txt; cat gpurun_out/ll_c5_$r.txt | cut -c1-160
done
