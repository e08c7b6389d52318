#!/bin/bash
# What the driver runs at round end on one GPU: build, pytest -m gpu, smoke(), the default bench line.
SHA=${1:-unknown}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
(echo "HEAD=$SHA"; timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider) > gpurun_out/pytest_driverlike.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_driverlike.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 400 python bench.py > gpurun_out/bench_driverlike.json 2> gpurun_out/bench_driverlike.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_driverlike.json'));r=d['roofline'];print(round(d['value']), round(d['e2e']['value']), r['bound'], round(r['frac'],3), r.get('isolated_frac'), d['gpu_launches'], d['clocks'])"
