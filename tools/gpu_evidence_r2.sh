#!/bin/bash
# Round-2 evidence run (one gpurun call): GPU tests, smoke, the default bench line (cfg2 +
# per_config cfg3/4/5, e2e, cpu_baseline, library_baseline), one bench line per other workload,
# the ncu launch list of the default bench command, and one `ncu --set full` capture per
# workload's kernel (full BASELINE batch) summarised on the box (tools/ncu_summary.py;
# per-launch DRAM traffic into gpurun_out/traffic.json).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; O=gpurun_out
: > $O/ev_status.txt
{ nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv; nproc; lscpu | grep "Model name"; } > $O/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/ev_status.txt
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/ev_status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/ev_status.txt
for c in ${CONFIGS:-1 3 4 5 6 7 8}; do
  timeout 900 python bench.py --config $c --no-e2e > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "bench cfg$c rc=$?" >> $O/ev_status.txt
done
CMD="python bench.py --steps 10 --warmup 3"
timeout 900 $CMD > $O/launch_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(reg|grp|blk|dmma|lane|generic|solve|nh|base|fxp)" -c 1000 --csv --log-file $O/launches.csv \
  $CMD > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> $O/ev_status.txt
cp profiles/traffic.json $O/traffic_in.json
for c in ${NCU_CONFIGS:-2 3 4 5}; do
  PC="python bench.py --config $c --per-config '' --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
  eval timeout 900 $PC > $O/ncu_plain_cfg$c.json 2>&1 && \
  eval timeout 1500 ncu --set full -f --clock-control none --import-source on -k regex:"k_" -s 3 -c 1 -o /tmp/prof_cfg$c $PC > $O/ncu_full_cfg$c.log 2>&1; echo "ncu full cfg$c rc=$?" >> $O/ev_status.txt
  K=$(python -c "import json; d=json.loads(open('$O/ncu_plain_cfg$c.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel'], d['batch_per_rank'])" 2>/dev/null)
  python tools/ncu_summary.py /tmp/prof_cfg$c.ncu-rep $O/summary_cfg$c.txt --traffic cfg$c ${K##* } ${K%% *} > /dev/null 2>&1
  ncu -i /tmp/prof_cfg$c.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $O/source_cfg$c.csv.gz
done
cp profiles/traffic.json $O/traffic.json
echo done >> $O/ev_status.txt
