python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do
for cfg in "POSEIDON_K1_RW=0" "POSEIDON_K1_RW=1" "POSEIDON_K1_RW=1 POSEIDON_K1_RWS=4" "POSEIDON_K1_RW=0 POSEIDON_K1_CFG=c"; do
  env $cfg timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('$cfg', round(d['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['isolated_kernel_ms']*1e3,1), round(r['pack']['ms_per_step']*1e3,1), round(d['sync_total_ms'],3))"
done; done
