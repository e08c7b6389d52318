#!/bin/bash
for shape in "4096 9216 256 1" "4096 9216 256 8"; do
  for c in a b; do
    echo -n "mode=W-only cfg=$c  "; POSEIDON_K1_MODE=1 POSEIDON_K1_CFG=$c python tools/k1_run.py $shape 10
    echo -n "mode=full   cfg=$c  "; POSEIDON_K1_CFG=$c python tools/k1_run.py $shape 10
  done
done
