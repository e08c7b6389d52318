#!/bin/bash
# Round-2 multi-GPU evidence (gpurun --gpus 4 -- bash tools/round2_check.sh SHA): GPU tests (incl. the
# 2- and 4-GPU parity script), the parity script's own log at 2 and 4 GPUs, bench lines at 1 / 2 / 4 GPUs,
# collective bus bandwidth.  Logs -> gpurun_out/.
SHA=${1:-unknown}
NG=$(nvidia-smi -L | wc -l)
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
(echo "HEAD=$SHA GPUs=$NG"; timeout -s KILL 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider) > gpurun_out/pytest_gpu_r2.log 2>&1
POSEIDON_K1_PROF=1 CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python tools/k1_prof.py > gpurun_out/k1_prof_r2.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 120 python tools/peaks.py > gpurun_out/peaks_r2.json 2> gpurun_out/peaks_r2.err
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r2.log
for P in 2 4; do
  [ "$NG" -ge "$P" ] || continue
  (echo "HEAD=$SHA P=$P"; timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P \
     --master-addr 127.0.0.1 --master-port $((29800 + P)) tests/mp_sync_check.py) > gpurun_out/mp_parity_r2_p$P.log 2>&1
  echo "mp P=$P rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py > gpurun_out/bench_r2_n1.json 2> gpurun_out/bench_r2_n1.err; echo "bench1 rc=$?"
for P in 2 4; do
  [ "$NG" -ge "$P" ] || continue
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
    --master-port $((29820 + P)) bench.py --gpus $P > gpurun_out/bench_r2_n$P.json 2> gpurun_out/bench_r2_n$P.err
  echo "bench$P rc=$?"
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
    --master-port $((29840 + P)) bench.py --gpus $P --override fc8=ps --no-cpu-baseline \
    > gpurun_out/bench_r2_n${P}_fc8ps.json 2> gpurun_out/bench_r2_n${P}_fc8ps.err
  echo "bench$P fc8=ps rc=$?"
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
    --master-port $((29860 + P)) tools/collective_bench.py > gpurun_out/collectives_r2_p$P.jsonl 2> gpurun_out/collectives_r2_p$P.err
  echo "coll$P rc=$?"
done
