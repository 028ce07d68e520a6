# Round-2 evidence: the headline kernel's ncu capture + the bench command's launch
# list, the EE graphs' launch lists, the decode launch lists, the GEMM table.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 50 --warmup 3 --no-extra --no-cpu-baseline --no-replicas > gpurun_out/r02_bench_under_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_diag3 -s 5 -c 1 -o gpurun_out/r02_k_diag3 -f python tools/profile_sweep.py diagonal 8 > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python tools/bench_ramp.py > gpurun_out/r02_micro_bench_ramp.txt 2>&1; echo "ramp rc=$?"
timeout 900 python tools/bench_gemm3.py > gpurun_out/r02_gemm3_vs_cublas.jsonl 2>&1; echo "gemm3 rc=$?"
for c in 1 2 3; do
  for r in vanilla ee; do
    timeout 600 ncu --nvtx --nvtx-include "$r/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_ll_c${c}_$r.csv python tools/profile_ee_graph.py $c > /dev/null 2>&1; echo "ncu c$c $r rc=$?"
    python tools/launch_list_summary.py gpurun_out/r02_ll_c${c}_$r.csv 30 > gpurun_out/r02_ll_c${c}_$r.txt
  done
done
for r in vanilla ee; do
  timeout 600 ncu --nvtx --nvtx-include "$r/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_ll_c5_$r.csv python tools/profile_gen.py > /dev/null 2>&1; echo "ncu c5 $r rc=$?"
  python tools/launch_list_summary.py gpurun_out/r02_ll_c5_$r.csv 20 > gpurun_out/r02_ll_c5_$r.txt
done
