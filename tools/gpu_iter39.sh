mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_convnet_gpu.py tests/test_gemm_tc_gpu.py -q -x -m gpu > gpurun_out/pt_iter.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 gpurun_out/pt_iter.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_ee_parity_gpu.py tests/test_ee_infer_gpu.py -q -x -m gpu > gpurun_out/pt_iter2.log 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/pt_iter2.log
timeout 900 python tools/bench_ee.py > gpurun_out/bench_ee.log 2>&1; echo "bench_ee rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/bench_ee.log'):
    if not l.startswith('{'): continue
    d = json.loads(l)
    print(d['config'], {k: round(d[k]['samples_per_s']) for k in d if isinstance(d[k], dict) and 'samples_per_s' in d[k]})
PY
timeout 600 ncu --nvtx --nvtx-include "vanilla/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_ll_c3_vanilla.csv python tools/profile_ee_graph.py 3 > /dev/null 2>&1; echo "ncu c3 rc=$?"
python tools/launch_list_summary.py gpurun_out/r02_ll_c3_vanilla.csv 30 > gpurun_out/r02_ll_c3_vanilla.txt; head -8 gpurun_out/r02_ll_c3_vanilla.txt
