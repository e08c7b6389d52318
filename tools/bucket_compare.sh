#!/bin/bash
# PS layer buckets (f1) at N GPUs: 0 (per layer) vs 256 KB vs 1 MB buckets on C2/C3/C4
N=${1:-4}
for cfg in C2 C4 C3; do for kb in 0 256 1024; do
  echo -n "$cfg bucket_kb=$kb "
  if [ "$N" = "1" ]; then cmd="python bench.py"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29900 + RANDOM % 90)) bench.py"; fi
  timeout -s KILL 200 $cmd --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --config $cfg --bucket-kb $kb 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), 'img/s', 'ms/step', round(d['ms_per_step'],3), 'exposed', round(d['exposed_sync_ms'],3), 'sync_total', round(d['sync_total_ms'],3))"
done; done
