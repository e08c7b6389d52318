# decomposition of K1 in the HBM regime (fc6, P*K = 256 and 512): full / W only / no W / MMA without TMEM loads
for shp in "4096 9216 256 1" "4096 9216 256 2"; do
  for mode in 0 1 7 6; do
    POSEIDON_K1_MODE=$mode timeout 60 python tools/k1_run.py $shp 30 | sed "s/^/mode$mode /"
  done
done
