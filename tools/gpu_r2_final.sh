# Final round-2 check: GPU tests, smoke, the default bench line, cfg7 and cfg9 lines, ncu of cfg7
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out
: > $O/fin_status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/fin_status.txt
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/fin_status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/fin_status.txt
for c in 7 9; do timeout 900 python bench.py --config $c --no-e2e > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "bench cfg$c rc=$?" >> $O/fin_status.txt; done
PC="python bench.py --config 7 --per-config '' --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
eval timeout 900 ncu --set full -f --clock-control none --import-source on -k regex:"k_" -s 3 -c 1 -o /tmp/prof_cfg7 $PC > $O/ncu_full_cfg7.log 2>&1; echo "ncu cfg7 rc=$?" >> $O/fin_status.txt
python tools/ncu_summary.py /tmp/prof_cfg7.ncu-rep $O/summary_cfg7.txt > /dev/null 2>&1
echo done >> $O/fin_status.txt
