#!/bin/bash
# Round-2 extra evidence on 4 GPUs: K1 configuration in the step at N = 2 / 4, the E10-style ablation on C3 and C4
# at 4 GPUs, and every layer's sync in isolation against its roofline at P = 1 / 2 / 4.  Logs -> gpurun_out/.
SHA=${1:-unknown}
python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/k1_cfg_multi.sh > gpurun_out/k1_cfg_multi.txt 2>&1; echo "k1 cfg rc=$?"
(echo "HEAD=$SHA"; for cfg in C3 C4; do for v in "--scheme ps --dwbp off" "--scheme ps" "--dwbp off" ""; do
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 300)) bench.py --gpus 4 --config $cfg $v --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads([l for l in open('/tmp/b.json') if l.startswith('{')][0]);print('$cfg [$v]', round(d['value']), round(d['exposed_sync_ms'],3), round(d['sync_total_ms'],3))"
done; done) > gpurun_out/ablation_r2.txt 2>&1; echo "ablation rc=$?"
for P in 1 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$P --master-addr 127.0.0.1 \
    --master-port $((29400 + P)) tools/layer_roofline.py > gpurun_out/layer_roofline_r2_p$P.jsonl 2> gpurun_out/layer_roofline_r2_p$P.err
  echo "layer roofline P=$P rc=$?"
done
