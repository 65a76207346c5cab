#!/bin/bash
# SURVEY 8(f) f3 on B200 where compute can matter: the cfg2 matrices (n = 8, c64) at an
# L2-resident batch (2^16: ~53 MB of A + X), each step replayed from a CUDA graph, for the
# proposed method and the paper's two existing methods.  Outputs gpurun_out/f3_*.json.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for bt in 65536 16384; do
  for m in proposed eqsolve trimat; do
    timeout 300 python bench.py --config 2 --batch $bt --inv-method $m --graph on --steps 400 --no-e2e --no-cpu-baseline --no-library > gpurun_out/f3_${m}_$bt.json 2>&1
  done
done
