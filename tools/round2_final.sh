#!/bin/bash
# Round-2 evidence on the final tree (gpurun --gpus 4 -- bash tools/round2_final.sh SHA): GPU tests, the
# multi-GPU parity script's logs at 2 / 4 GPUs, default bench lines at 1 / 2 / 4 GPUs, C2 at 1 / 2 / 4, C4 and
# the E10-style ablation (C3, C4) at 4, the N = 1 launch list and an ncu --set full capture of K1.
SHA=${1:-unknown}
NG=$(nvidia-smi -L | wc -l)
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
(echo "HEAD=$SHA GPUs=$NG (test_gpu_multi deselected here: the same script runs below with its own logs)"
 timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -k "not test_multi_gpu_sync" -p no:cacheprovider) > gpurun_out/pytest_gpu_final.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_final.log
for P in 2 4; do
  [ "$NG" -ge "$P" ] || continue
  (echo "HEAD=$SHA P=$P"; timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P \
     --master-addr 127.0.0.1 --master-port $((29700 + P)) tests/mp_sync_check.py) > gpurun_out/mp_parity_final_p$P.log 2>&1
  echo "mp P=$P rc=$?"; grep -c MP_OK gpurun_out/mp_parity_final_p$P.log
done
run() {  # name P args...
  local name=$1 P=$2; shift 2
  if [ "$P" = 1 ]; then
    CUDA_VISIBLE_DEVICES=0 timeout -s KILL 400 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  else
    timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
      --master-port $((29750 + RANDOM % 200)) bench.py --gpus $P "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  fi
  echo "bench $name rc=$?"
}
run n1 1
for P in 2 4; do [ "$NG" -ge "$P" ] && run n$P $P; done
for P in 1 2 4; do [ "$NG" -ge "$P" ] && run c2_n$P $P --config C2 --no-cpu-baseline; done
if [ "$NG" -ge 4 ]; then
  run c4_n4 4 --config C4 --no-cpu-baseline
  for cfg in C3 C4; do
    run abl_${cfg}_psoff 4 --config $cfg --scheme ps --dwbp off --graph off --no-cpu-baseline --no-e2e
    run abl_${cfg}_pson 4 --config $cfg --scheme ps --graph off --no-cpu-baseline --no-e2e
    run abl_${cfg}_sacpoff 4 --config $cfg --dwbp off --graph off --no-cpu-baseline --no-e2e
    run abl_${cfg}_sacpon 4 --config $cfg --graph off --no-cpu-baseline --no-e2e
  done
fi
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 ncu --nvtx --nvtx-include "timed" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
echo "ncu launches rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:recon_tcgen05_2sm --launch-skip 5 \
  --launch-count 1 -o gpurun_out/k1_final python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
echo "ncu k1 rc=$?"
for f in gpurun_out/bench_*.json; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][0])
    r = d["roofline"]
    print(f.split("bench_")[1][:-5], d["n_gpus"], round(d["value"]), round(d["e2e"]["value"]) if d.get("e2e") else None,
          round(d["ms_per_step"], 3), "exposed", round(d["exposed_sync_ms"], 4), "sync", round(d["sync_total_ms"], 3),
          r["bound"], round(r["frac"], 3), d["details"].get("cuda_graph"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(f, "ERR", e)
PY
done
