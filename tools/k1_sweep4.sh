#!/bin/bash
./tools/w_stream_probe_s3 | head -1; ./tools/w_stream_probe_s5 | head -1; ./tools/w_stream_probe | head -1
for c in a b c; do for m in 0 1; do
  echo -n "cfg=$c mode=$m "; POSEIDON_K1_MODE=$m POSEIDON_K1_CFG=$c python tools/k1_run.py 4096 9216 256 1 10
done; done
for c in b c; do echo -n "cfg=$c P=2 "; POSEIDON_K1_CFG=$c python tools/k1_run.py 4096 9216 256 2 10; done
