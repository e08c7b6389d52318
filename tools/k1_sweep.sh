#!/bin/bash
# K1 config sweep (raster x stage/slot config) on the HBM- and tensor-bound fc6 shapes
for shape in "4096 9216 256 1" "4096 9216 256 2" "4096 9216 256 8" "1000 4096 256 1" "4096 4096 256 1"; do
  for r in m n; do for c in a b; do
    echo -n "raster=$r cfg=$c  "; POSEIDON_K1_RASTER=$r POSEIDON_K1_CFG=$c python tools/k1_run.py $shape 10
  done; done
done
