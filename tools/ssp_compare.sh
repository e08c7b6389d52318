#!/bin/bash
# BSP (s = 0) vs SSP (s = 1) at N GPUs on C2/C3/C4 (paper E11)
N=${1:-4}
for cfg in C2 C3 C4; do for ssp in 0 1; do
  echo -n "$cfg ssp=$ssp "
  if [ "$N" = "1" ]; then cmd="python bench.py"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29900 + RANDOM % 90)) bench.py"; fi
  timeout -s KILL 200 $cmd --gpus $N --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --config $cfg --ssp $ssp 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), 'img/s', 'ms/step', round(d['ms_per_step'],3), 'exposed', round(d['exposed_sync_ms'],3), 'sync_total', round(d['sync_total_ms'],3))"
done; done
