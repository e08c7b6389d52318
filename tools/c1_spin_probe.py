"""C1 timing probe: bench.c1_step under two device-spin lengths (the spin must outlast the host enqueue of
the call for the events to time the GPU work only)."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_1512_06216_b200 as pz
dev = torch.device("cuda", 0)
for spin in ("2000000", "10000000"):
    os.environ["C1_SPIN_CYCLES"] = spin
    r = bench.c1_step(pz, dev)
    print(spin, json.dumps({k: v for k, v in r.items() if k.startswith(("gpu", "call"))}), flush=True)
