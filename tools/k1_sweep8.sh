# K1 HBM regime (fc6, P*K=256): stage / W-slot split x decomposition mode
#   cfg 0 <3,8>  1 <4,5> (production)  2 <2,8>  3 <5,4>;  mode 0 full, 1 W stream only, 7 no W traffic
for cfg in a b c d; do for mode in 0 1 7; do
  POSEIDON_K1_CFG=$cfg POSEIDON_K1_MODE=$mode timeout -s KILL 60 python tools/k1_run.py 4096 9216 256 1 30 | sed "s/^/cfg=$cfg mode=$mode /"
done; done
