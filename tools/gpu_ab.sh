#!/bin/bash
# A/B timing: default build vs libhpdinv_<variant>.so for the configs in $CONFIGS.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; O=gpurun_out
: > $O/status.txt
if [ -n "$PYTEST_K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$PYTEST_K" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
fi
for c in ${CONFIGS:-2 3}; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/b_base_cfg$c.json 2>&1
  for v in ${VARIANTS}; do
    HPDINV_LIB=$PWD/paper_1111_4144_b200/libhpdinv_$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/b_${v}_cfg$c.json 2>&1
  done
done
echo done >> $O/status.txt
