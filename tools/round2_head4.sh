#!/bin/bash
# Short final-tree check on a 4-GPU box (gpurun --gpus 4 -- bash tools/round2_head4.sh SHA): every GPU test
# (test_gpu_multi runs tests/mp_sync_check.py at 2 and 4 ranks), then the default bench lines at 1 / 2 / 4 GPUs
# and C2 at 4.
SHA=${1:-unknown}
(echo "HEAD=$SHA GPUs=$(nvidia-smi -L | wc -l)"; timeout -s KILL 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider) \
  > gpurun_out/pytest_gpu_head4.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_head4.log
run() {  # name P args...
  local name=$1 P=$2; shift 2
  if [ "$P" = 1 ]; then
    CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py "$@" > gpurun_out/bench_head_$name.json 2> gpurun_out/bench_head_$name.err
  else
    timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
      --master-port $((29750 + RANDOM % 200)) bench.py --gpus $P "$@" > gpurun_out/bench_head_$name.json 2> gpurun_out/bench_head_$name.err
  fi
  echo "bench $name rc=$?"
}
run n1 1
run n2 2
run n4 4
run c2_n4 4 --config C2 --no-cpu-baseline
