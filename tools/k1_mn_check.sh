#!/bin/bash
# K1 MN-major operands (round 2): A/B against the K-major kernel on the same factors (speed, W digests).
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
: > gpurun_out/k1_mn.txt
for cfg in "K1_AB_MN=0" "K1_AB_MN=1" "K1_AB_MN=1 POSEIDON_K1_RW=0" "K1_AB_MN=1 POSEIDON_K1_RW=1"; do
  env $cfg timeout -s KILL 120 python tools/k1_ab.py >> gpurun_out/k1_mn.txt 2>&1; echo "$cfg rc=$?" >> gpurun_out/k1_mn.txt
done
cat gpurun_out/k1_mn.txt
