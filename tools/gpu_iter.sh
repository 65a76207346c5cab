#!/bin/bash
# Iteration GPU call: GPU tests (optionally filtered), per-config bench lines, and an ncu
# --set full capture of one config's kernel.  Env: PYTEST_K (pytest -k filter, "" = all),
# CONFIGS (bench configs, default "2 3"), NCU_CFG (config to profile, "" = none),
# NCU_KERNEL (regex of the kernel name).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
: > $O/status.txt
if [ "${PYTEST_K-x}" != "skip" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
fi
for c in ${CONFIGS:-2 3}; do
  timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "bench cfg$c rc=$?" >> $O/status.txt
done
if [ -n "$NCU_CFG" ]; then
  CMD="python bench.py --config $NCU_CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 900 $CMD > $O/ncu_plain.json 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNEL:-k_}" -s 3 -c 1 -o $O/prof_cfg$NCU_CFG $CMD > $O/ncu_full.log 2>&1
  echo "ncu rc=$?" >> $O/status.txt
fi
