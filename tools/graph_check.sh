#!/bin/bash
# CUDA-graph step capture (round 2): GPU test, then C2 / C3 bench lines with and without the graph.
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python -m pytest tests/test_gpu_graph.py -x -q -p no:cacheprovider 2>&1 | tail -15
for cfg in C2 C3; do for gr in off on; do
  timeout -s KILL 300 python bench.py --config $cfg --graph $gr --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err; echo "rc=$?"; tail -2 /tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));r=d['roofline'];print('$cfg graph $gr', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], round(d['exposed_sync_ms'],4), round(d['sync_total_ms'],4), round(r['frac'],3), d['gpu_launches'])"
done; done
