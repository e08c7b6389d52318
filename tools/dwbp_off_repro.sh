python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
for a in "--dwbp off" "--dwbp off --factors pack" "" ; do
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py $a --no-cpu-baseline --no-e2e --steps 10 > /tmp/d.json 2> /tmp/d.err; echo "n1 [$a] rc=$?"
python -c "import json;d=json.load(open('/tmp/d.json'));print(round(d['value']), d['exposed_sync_ms'], d['sync_total_ms'], d['details']['factors'])"
done
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --dwbp off --no-cpu-baseline --no-e2e --steps 10 > /tmp/d2.json 2> /tmp/d2.err; echo "n2 rc=$?"
python -c "import json;d=json.loads([l for l in open('/tmp/d2.json') if l.startswith('{')][0]);print(round(d['value']), d['exposed_sync_ms'], d['sync_total_ms'])"
