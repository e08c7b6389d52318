#!/bin/bash
# K1 RW-epilogue check (round 2, 1 GPU): W register-path probe, K1 A/B of the W ring vs the RW epilogue
# (speed + bit-identical W digests), then the GPU tests.  Logs -> gpurun_out/.
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/w_reg_probe tools/w_reg_probe.cu && timeout -s KILL 120 /tmp/w_reg_probe > gpurun_out/w_reg_probe.txt 2>&1
cat gpurun_out/w_reg_probe.txt
: > gpurun_out/k1_ab.txt
for cfg in "POSEIDON_K1_RW=0" "POSEIDON_K1_RWD=2" "POSEIDON_K1_RWD=3" "POSEIDON_K1_RWD=4" "POSEIDON_K1_RWS=4" "POSEIDON_K1_RWS=5"; do
  env $cfg timeout -s KILL 120 python tools/k1_ab.py >> gpurun_out/k1_ab.txt 2>&1; echo "$cfg rc=$?" >> gpurun_out/k1_ab.txt
done
cat gpurun_out/k1_ab.txt
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_rw.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_rw.log
timeout -s KILL 300 python bench.py --no-cpu-baseline > gpurun_out/bench_rw.json 2> gpurun_out/bench_rw.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_rw.json'));r=d['roofline'];print(d['value'],d['e2e']['value'],r['frac'],r['kernel_ms'],r.get('isolated_kernel_ms'),r.get('isolated_frac'))"
