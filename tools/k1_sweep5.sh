#!/bin/bash
for m in 0 1; do for eg in 2 1; do for wp in 0 1; do
  echo -n "mode=$m epi=$eg wpol=$wp "; POSEIDON_K1_MODE=$m POSEIDON_K1_EPI=$eg POSEIDON_K1_WPOL=$wp python tools/k1_run.py 4096 9216 256 1 10
done; done; done
