#!/bin/bash
# Round-2 multi-GPU evidence on the final tree (gpurun --gpus 4 -- bash tools/round2_final.sh SHA): GPU tests
# (incl. the 2- and 4-GPU parity script), the parity script's own logs, default bench lines at 1 / 2 / 4 GPUs,
# C2 with and without the CUDA-graph step at 1 / 2 / 4 GPUs, C4 at 4 GPUs.  Logs -> gpurun_out/.
SHA=${1:-unknown}
NG=$(nvidia-smi -L | wc -l)
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
(echo "HEAD=$SHA GPUs=$NG"; timeout -s KILL 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider) > gpurun_out/pytest_gpu_final.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_final.log
for P in 2 4; do
  [ "$NG" -ge "$P" ] || continue
  (echo "HEAD=$SHA P=$P"; timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P \
     --master-addr 127.0.0.1 --master-port $((29700 + P)) tests/mp_sync_check.py) > gpurun_out/mp_parity_final_p$P.log 2>&1
  echo "mp P=$P rc=$?"
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
for P in 1 2 4; do
  [ "$NG" -ge "$P" ] || continue
  run c2_graph_n$P $P --config C2 --no-cpu-baseline
  run c2_eager_n$P $P --config C2 --graph off --no-cpu-baseline
done
[ "$NG" -ge 4 ] && run c4_n4 4 --config C4 --no-cpu-baseline
[ "$NG" -ge 4 ] && run c3_graph_n4 4 --graph on --no-cpu-baseline
for f in gpurun_out/bench_*.json; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][0])
    r = d["roofline"]
    print(f.split("bench_")[1][:-5], d["n_gpus"], round(d["value"]), round(d["e2e"]["value"]) if d.get("e2e") else None,
          round(d["ms_per_step"], 3), "exposed", round(d["exposed_sync_ms"], 4), "sync", round(d["sync_total_ms"], 3),
          r["bound"], round(r["frac"], 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
except Exception as e:
    print(f, "ERR", e)
PY
done
