python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "mn or inplace or alexnet" 2>&1 | tail -3
for cfg in "K1_AB_MN=0" "K1_AB_MN=1 POSEIDON_K1_MN4=0" "K1_AB_MN=1 POSEIDON_K1_MN4=1"; do env $cfg timeout -s KILL 120 python tools/k1_ab.py 2>&1 | head -5; done
for ip in on off on off; do
  timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --inplace $ip > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('inplace $ip', round(d['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['isolated_kernel_ms']*1e3,1), round(r['pack']['ms_per_step']*1e3,1), round(d['sync_total_ms'],3))"
done
