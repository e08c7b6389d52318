python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29811 tests/mp_sync_check.py > gpurun_out/mp2_async.log 2>&1; echo "mp rc=$?"; tail -12 gpurun_out/mp2_async.log
for f in pack async; do
timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29822 bench.py --gpus 2 --no-cpu-baseline --no-e2e --factors $f > /tmp/b2.json 2>/dev/null
python -c "import json;d=json.loads([l for l in open('/tmp/b2.json') if l.startswith('{')][0]);r=d['roofline'];print('$f', round(d['value']), round(r['frac'],3), round(r['kernel_ms']*1e3,1), round(r['pack']['ms_per_step']*1e3,1), round(d['sync_total_ms'],3), round(d['exposed_sync_ms'],3))"
done
