#!/bin/bash
# Regression demo for the round-1 race in the fused NVLS PS kernel:
#   1. copy the repo to /tmp, put the round-1 gradient clear back (block j clears its grid-strided share
#      of the WHOLE padded buffer, including other owners' shards), build, run mp_sync_check check 10
#      under the in-kernel CTA fuzz -> expected to FAIL (lost gradient contributions);
#   2. run the same check on this tree (the fix: block j clears only what block j of every rank
#      reduced) -> expected to PASS.
# Usage (GPU box, >= 2 GPUs): bash tools/nvls_race_demo.sh [nproc] [fuzz_us]
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NP=${1:-2}
FZ=${2:-200}
OUT=${OUT:-$ROOT/gpurun_out}
mkdir -p "$OUT"
LEG=/tmp/poseidon_legacy_zero
rm -rf "$LEG" && mkdir -p "$LEG"
(cd "$ROOT" && tar --exclude=./gpurun_out --exclude=./build --exclude='*.so' -cf - .) | (cd "$LEG" && tar xf -)
python - "$LEG/paper_1512_06216_b200/csrc/k_ps_nvls.cu" <<'PY'
import sys
p = sys.argv[1]
s = open(p).read()
fixed = """    for (int q = 0; q < nranks; ++q)
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s4; i += stride) gl[q * s4 + i] = z;"""
legacy = """    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nranks * s4; i += stride) gl[i] = z;"""
assert fixed in s, "fixed clear loop not found"
open(p, "w").write(s.replace(fixed, legacy))
print("patched", p, "back to the round-1 clear")
PY
(cd "$LEG" && python paper_1512_06216_b200/build.py --force) || exit 1
run() {
  local dir=$1 tag=$2
  (cd "$dir" && POSEIDON_FUZZ_US=$FZ timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$NP" \
     --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) tests/mp_sync_check.py --race-only) \
     > "$OUT/nvls_race_${tag}_p${NP}.log" 2>&1
  echo "$tag: exit $?"
}
run "$LEG" legacy
run "$ROOT" fixed
