#!/bin/bash
# Round-end evidence run: GPU tests, the default bench line (cfg2, e2e + cpu_baseline), one bench
# line per other config, the ncu launch list of the default bench command, and one
# `ncu --set full` capture per config's kernel.  Outputs under gpurun_out/ (summarise into profiles/).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; O=gpurun_out
: > $O/ev_status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/ev_status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/ev_status.txt
for c in ${CONFIGS:-3 4 5}; do
  timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "bench cfg$c rc=$?" >> $O/ev_status.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/ev_status.txt
for c in ${NCU_CONFIGS:-2 3 4 5}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 3 -c 1 -o $O/prof_cfg$c \
    python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full_cfg$c.log 2>&1; echo "ncu full cfg$c rc=$?" >> $O/ev_status.txt
done
