#!/bin/bash
# One-GPU evidence for the current tree (gpurun -- bash tools/gpu1_check.sh SHA): build, GPU tests, the bench
# line, the NVTX-filtered launch list and ncu --set full captures of K1 (fc6) and K3 from the bench.
SHA=${1:-unknown}
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
(echo "HEAD=$SHA"; timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider) > gpurun_out/pytest_gpu1.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu1.log
timeout -s KILL 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
cat gpurun_out/bench_n1.json
timeout -s KILL 600 ncu --nvtx --nvtx-include "timed" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
echo "ncu launches rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:recon_tcgen05_2sm --launch-skip 5 \
  --launch-count 1 -o gpurun_out/k1_bench python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
echo "ncu k1 rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:pack_uv --launch-skip 6 \
  --launch-count 3 -o gpurun_out/k3_bench python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k3.log 2>&1
echo "ncu k3 rc=$?"
