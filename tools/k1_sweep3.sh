#!/bin/bash
shape="4096 9216 256 1"
for m in 1 2 3; do for c in a b; do
  echo -n "mode=$m cfg=$c  "; POSEIDON_K1_MODE=$m POSEIDON_K1_CFG=$c python tools/k1_run.py $shape 10
done; done
python - <<'PY'
import torch
n=4096*9216
a=torch.randn(n,device='cuda'); b=torch.empty_like(a)
s,e=torch.cuda.Event(True),torch.cuda.Event(True)
for name,fn in [("copy",lambda: b.copy_(a)),("read-sum",lambda: a.sum()),("fill",lambda: b.fill_(1.0))]:
    for _ in range(3): fn()
    s.record(); [fn() for _ in range(10)]; e.record(); e.synchronize()
    ms=s.elapsed_time(e)/10
    by = 2*4*n if name=="copy" else 4*n
    print(f"torch {name}: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s")
PY
