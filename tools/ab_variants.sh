#!/bin/bash
# A/B timing of variant builds (paper_1111_4144_b200/libhpdinv_<v>.so, built with
# `python paper_1111_4144_b200/_build.py --variant <v> -D...`).  Env: VARIANTS, CONFIGS.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
: > gpurun_out/ab_status.txt
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then L=paper_1111_4144_b200/libhpdinv.so; else L=paper_1111_4144_b200/libhpdinv_$v.so; fi
  for c in ${CONFIGS:-4 5}; do
    HPDINV_LIB=$PWD/$L timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_cfg$c.json 2>gpurun_out/ab_${v}_cfg$c.err
    echo "$v cfg$c rc=$?" >> gpurun_out/ab_status.txt
  done
done
