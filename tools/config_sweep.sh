#!/bin/bash
# Run every BASELINE config (and the C3 ablations) once on the visible GPUs; one JSON line each.
N=${1:-1}
run() {
  if [ "$N" = "1" ]; then python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@";
  else python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 10 --warmup 3 --no-e2e "$@"; fi
}
for cfg in C2 C3 C4 C5; do echo "== $cfg"; run --config $cfg 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(json.dumps({k:d[k] for k in ('value','ms_per_step','exposed_sync_ms','sync_total_ms','nccl_bytes_sent_per_iter')}), r['kernel'], round(r['frac'],3), r['bound'])"; done
echo "== C3 dwbp off";  run --config C3 --dwbp off 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['exposed_sync_ms'], d['sync_total_ms'])"
echo "== C3 all-PS";    run --config C3 --scheme ps 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['exposed_sync_ms'], d['sync_total_ms'])"
echo "== C3 all-PS dwbp off"; run --config C3 --scheme ps --dwbp off 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['exposed_sync_ms'], d['sync_total_ms'])"
