#!/bin/bash
# K1 ring configuration sweep inside the C3 step at P = 1 (round 2): images/s, in-step K1 frac / us, isolated us,
# per configuration (POSEIDON_K1_CFG), twice; then the MN-major tcgen05 probe.
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do
for c in b c h e f g; do
  POSEIDON_K1_RW=0 POSEIDON_K1_CFG=$c timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('cfg $c', round(d['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['isolated_kernel_ms']*1e3,1), round(d['sync_total_ms'],3))"
done; done
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_probe_mn tools/tc_probe_mn.cu && timeout -s KILL 60 /tmp/tc_probe_mn | grep -v "nonzero 0$" > gpurun_out/tc_probe_mn2.txt 2>&1; grep -c "" gpurun_out/tc_probe_mn2.txt; grep "SW128_32B" gpurun_out/tc_probe_mn2.txt | head -40
