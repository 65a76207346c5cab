#!/bin/bash
# ncu --set full of configs' kernels (one ncu-tool call); summaries are produced on the box
# and the large reports are dropped unless KEEP_REP=1.  Env: CFGS (configs), KREGEX.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; O=gpurun_out; : > $O/status.txt
for c in $CFGS; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 900 $CMD > $O/plain_cfg$c.json 2>&1; echo "plain cfg$c rc=$?" >> $O/status.txt
done
for c in $CFGS; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_(cta|lane|reg)}" -s 2 -c 1 -o /tmp/prof_cfg$c $CMD > $O/ncu_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?" >> $O/status.txt
  python tools/ncu_summary.py /tmp/prof_cfg$c.ncu-rep $O/summary_cfg$c.txt > /dev/null 2>&1
  ncu -i /tmp/prof_cfg$c.ncu-rep --page source --csv --print-source sass > $O/source_cfg$c.csv 2>/dev/null
  gzip -f $O/source_cfg$c.csv
  [ "$KEEP_REP" = 1 ] && cp /tmp/prof_cfg$c.ncu-rep $O/
done
