#!/bin/bash
# C3 with / without the CUDA-graph step at N = 1 and 2 (round 2, after the priority launch attribute).
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do for gr in off on; do
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py --graph $gr --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('N=1 graph $gr', round(d['value']), round(d['e2e']['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(d['exposed_sync_ms'],4), round(d['sync_total_ms'],3))"
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 2 --graph $gr --no-cpu-baseline > /tmp/b2.json 2>/dev/null
  python -c "import json;d=json.loads([l for l in open('/tmp/b2.json') if l.startswith('{')][0]);r=d['roofline'];print('N=2 graph $gr', round(d['value']), round(d['e2e']['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(d['exposed_sync_ms'],4), round(d['sync_total_ms'],3))"
done; done
