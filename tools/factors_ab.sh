#!/bin/bash
# SFB factor paths in the C3 step at P = 1 (round 2): async pack / MN in place / round-1 pack, twice each;
# GPU tests first.  (bench.py --factors)
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_fac.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fac.log
for rep in 1 2; do for f in async mn pack; do
  timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --factors $f > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('$f', round(d['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['isolated_kernel_ms']*1e3,1), round(r['pack']['ms_per_step']*1e3,1), round(d['sync_total_ms'],3), round(d['exposed_sync_ms'],3))"
done; done
