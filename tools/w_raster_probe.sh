#!/bin/bash
# W-stream probe: tile raster x box shape x slots (round 2; does DRAM locality cap the smem-ring stream?)
for S in 5 6; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSLOTS_=$S -o /tmp/wsp$S tools/w_stream_probe.cu -lcuda || exit 1
  for R in 0 1 2; do RASTER=$R timeout -s KILL 60 /tmp/wsp$S; done
done
