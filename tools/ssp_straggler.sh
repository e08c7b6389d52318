#!/bin/bash
# BSP vs SSP s=1 with an injected straggler (one pseudo-random rank delayed D us per step), N GPUs
N=${1:-4}
for cfg in C3 C2; do for D in 0 1000 3000; do for ssp in 0 1; do
  echo -n "$cfg straggle_us=$D ssp=$ssp "
  timeout -s KILL 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29900 + RANDOM % 90)) bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --config $cfg --ssp $ssp --straggle-us $D 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value']), 'img/s', 'ms/step', round(d['ms_per_step'],3), 'exposed', round(d['exposed_sync_ms'],3))"
done; done; done
