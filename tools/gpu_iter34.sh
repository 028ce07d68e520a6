# iteration: routed ResNet classifier; then refreshed launch lists (EE graphs, decode)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_convnet_gpu.py tests/test_ee_parity_gpu.py tests/test_ee_infer_gpu.py tests/test_heads_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt_iter.log
timeout 900 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/bench_ee.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print(d['config'], {k: round(d[k]['samples_per_s']) for k in d if isinstance(d[k], dict) and 'samples_per_s' in d[k]})
PY
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
