#!/bin/bash
# K1 at P*K = 512 (fc6 at 2 GPUs): every ring configuration and the RW epilogue alone (tools/k1_ab.py shapes 1-2).
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
for cfg in d i j; do
  POSEIDON_K1_RW=0 POSEIDON_K1_CFG=$cfg timeout -s KILL 120 python tools/k1_ab.py 2>&1 | sed -n 2,3p
done
POSEIDON_K1_RW=1 timeout -s KILL 120 python tools/k1_ab.py 2>&1 | sed -n 2,3p
