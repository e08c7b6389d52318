#!/bin/bash
# K1 configuration inside the C3 step at N = 2 and 4 (round 2): ring <5,4> (d) / <4,6> (g) / RW epilogue, twice.
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
NG=$(nvidia-smi -L | wc -l)
for P in 2 4; do
  [ "$NG" -ge "$P" ] || continue
  for rep in 1 2; do for cfg in "POSEIDON_K1_RW=0 POSEIDON_K1_CFG=d" "POSEIDON_K1_RW=0 POSEIDON_K1_CFG=g" "POSEIDON_K1_RW=1"; do
    env $cfg timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $P --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null
    python -c "import json;d=json.loads([l for l in open('/tmp/b.json') if l.startswith('{')][0]);r=d['roofline'];print('P=$P $cfg', round(d['value']), r['bound'], round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['isolated_kernel_ms']*1e3,1), round(d['sync_total_ms'],3), round(d['exposed_sync_ms'],3))"
  done; done
done
