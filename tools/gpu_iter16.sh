mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_distributed_gpu.py tests/test_gpu_parity.py -q -x -k "windows or two_rank" 2>&1 | tail -3
timeout 900 python bench.py --no-extra --no-cpu-baseline --no-replicas > gpurun_out/bench_w.log 2> gpurun_out/bench_w.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_w.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_w.log').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','gpu_launches','timed_as','headline_matches_single_sweep')})
print(d['roofline']['frac'], d['roofline']['achieved'])
print(d['graph_of_sweeps'])
print(d['clocks'])
PY
EEB200_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline --no-extra --no-replicas > gpurun_out/bench_n2.log 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"; tail -1 gpurun_out/bench_n2.log | cut -c1-300
