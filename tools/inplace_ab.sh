#!/bin/bash
# In-place factors (POSEIDON_FLAG_INPLACE_FACTORS) A/B in the C3 step at P = 1 (round 2), GPU tests, the launch
# list of the default (in-place) bench.
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_ip.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ip.log
for rep in 1 2; do for ip in on off; do
  timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --inplace $ip > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('inplace $ip', round(d['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['isolated_kernel_ms']*1e3,1), round(r['pack']['ms_per_step']*1e3,1), round(d['sync_total_ms'],3))"
done; done
timeout -s KILL 600 ncu --nvtx --nvtx-include "timed" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_ip.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
echo "ncu rc=$?"
