for P in 2 4; do for U in 2 4 8; do for G in 64 128 148 296; do
POSEIDON_NVLS_U=$U POSEIDON_NVLS_GRID=$G timeout -s KILL 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 --master-port $((29700+P+U*10+G)) tools/collective_bench.py --ps-only 2>&1 | grep "^{" ; done; done; done > gpurun_out/nvls_sweep.jsonl
