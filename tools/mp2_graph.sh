python paper_1512_06216_b200/build.py --force > gpurun_out/build.log 2>&1 || exit 1
MP_VERBOSE=1 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29811 tests/mp_sync_check.py --graph-only > gpurun_out/mp2_graph.log 2>&1; echo "rc=$?"
grep -v "^frame\|TCPStore\|^Exception" gpurun_out/mp2_graph.log | grep -v "replay\|captured" | head -30
timeout -s KILL 300 python -m pytest tests/test_gpu_graph.py -q -p no:cacheprovider 2>&1 | tail -2
