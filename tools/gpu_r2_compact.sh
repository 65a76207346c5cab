# A/B: k_grp COMPACT shared-memory layout (libhpdinv_compact.so) vs default at cfg3; GPU tests on the variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/compact; O=gpurun_out/compact
: > $O/status.txt
HPDINV_LIB=$PWD/paper_1111_4144_b200/libhpdinv_compact.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_compact.log 2>&1; echo "pytest compact rc=$?" >> $O/status.txt
B="--per-config '' --no-e2e --no-cpu-baseline --no-library"
km() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['roofline']['kernel_ms'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))" $1 2>&1; }
for rep in 1 2 3; do
  for v in base compact; do
    f=$O/c3_${v}_r$rep.json
    if [ $v = base ]; then eval timeout 300 python bench.py --config 3 $B > $f 2>/dev/null
    else eval HPDINV_LIB=$PWD/paper_1111_4144_b200/libhpdinv_compact.so timeout 300 python bench.py --config 3 $B > $f 2>/dev/null; fi
    km $f >> $O/status.txt
  done
done
M=gpu__time_duration.sum,launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,l1tex__t_sector_hit_rate.pct,launch__registers_per_thread
P="--per-config '' --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
eval HPDINV_LIB=$PWD/paper_1111_4144_b200/libhpdinv_compact.so timeout 300 ncu --metrics $M --clock-control none -k regex:k_grp -s 2 -c 1 --csv python bench.py --config 3 $P > $O/ncu_c3_compact.csv 2>/dev/null
echo done >> $O/status.txt
