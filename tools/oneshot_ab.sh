#!/bin/bash
# K2o one-shot small-layer PS sync (round 2): multi-GPU parity, then C2 / C4 with and without it (POSEIDON_ONESHOT).
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
NG=$(nvidia-smi -L | wc -l)
POSEIDON_ONESHOT=1 timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port 29811 tests/mp_sync_check.py > gpurun_out/mp_oneshot_p$NG.log 2>&1; echo "mp P=$NG rc=$?"
grep -c MP_OK gpurun_out/mp_oneshot_p$NG.log
for rep in 1 2; do for cfg in C2 C4; do for os in 1 0; do
  POSEIDON_ONESHOT=$os timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 300)) bench.py --gpus $NG --config $cfg --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads([l for l in open('/tmp/b.json') if l.startswith('{')][0]);print('$cfg oneshot=$os', round(d['value']), round(d['exposed_sync_ms'],4), round(d['sync_total_ms'],3), round(d['exposed_sync_ms']/d['sync_total_ms'],3))"
done; done; done
