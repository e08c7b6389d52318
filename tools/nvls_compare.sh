#!/bin/bash
# NCCL RS/K2/AG vs fused NVLS PS at N GPUs on C2/C3/C4
N=${1:-4}
for cfg in C2 C3 C4; do for nv in off on; do
  echo -n "$cfg nvls=$nv "
  timeout -s KILL 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --config $cfg --nvls $nv 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), 'img/s', 'exposed', round(d['exposed_sync_ms'],3), 'sync_total', round(d['sync_total_ms'],3), d['details']['ps_path'])"
done; done
