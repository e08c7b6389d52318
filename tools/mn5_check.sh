#!/bin/bash
# MN-major operand layouts after the encoder fix (round 2): K-major vs MN 3-D / 4-D boxes (MN4=2 was a 5-D probe, removed),
# digests and speed; then the GPU tests.
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
K1_AB_MN=0 timeout -s KILL 120 python tools/k1_ab.py 2>&1 | head -8
for m in 0 1 2; do K1_AB_MN=1 POSEIDON_K1_MN4=$m timeout -s KILL 120 python tools/k1_ab.py 2>&1 | head -8; done
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
