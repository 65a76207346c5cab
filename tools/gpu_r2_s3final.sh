# Session-3 closing check at HEAD: GPU tests, smoke, default bench line, cfg3 line, cfg3 ncu --set full
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/s3; O=gpurun_out/s3
: > $O/status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/status.txt
for c in 3 5; do timeout 600 python bench.py --config $c --no-library > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "bench cfg$c rc=$?" >> $O/status.txt; done
PC="python bench.py --config 3 --per-config '' --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
eval timeout 900 ncu --set full -f --clock-control none --import-source on -k regex:k_grp -s 3 -c 1 -o /tmp/prof_cfg3 $PC > $O/ncu_full_cfg3.log 2>&1; echo "ncu cfg3 rc=$?" >> $O/status.txt
python tools/ncu_summary.py /tmp/prof_cfg3.ncu-rep $O/summary_cfg3.txt > /dev/null 2>&1
echo done >> $O/status.txt
