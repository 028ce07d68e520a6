"""Data-parallel EE serving, one replica per GPU (paper_2312_05385_b200/replicas.py).

    python tools/bench_replicas.py [c1|c2|c3] [batches]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/bench_replicas.py c3 64

Rank 0 prints one JSON line: samples/s over all replicas (all requests ÷ the
slowest replica's CUDA-event time) and p50 batch latency."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

from paper_2312_05385_b200.replicas import run_replicas


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    agg = run_replicas(config, nb)
    if agg is not None:
        print(json.dumps(agg), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
