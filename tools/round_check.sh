# End-of-round evidence on a 4-GPU box (gpurun --gpus 4 -- bash tools/round_check.sh):
# GPU tests, bench lines at 1 / 2 / 4 GPUs with the defaults, the NVTX-filtered launch list of the 1-GPU bench
# and one ncu --set full capture of K1 (fc6) from it.  Summaries: tools/ncu_summary.py -> profiles/.
set -x
timeout -s KILL 1000 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo rc=$?
timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc=$?
timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo rc=$?
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 ncu --nvtx --nvtx-include "timed" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncu rc=$?
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:recon_tcgen05_2sm --launch-skip 5 --launch-count 1 -o gpurun_out/k1_bench python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncu2 rc=$?
