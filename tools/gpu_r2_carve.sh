# Carveout and L2 fetch-granularity experiments at cfg3 / cfg5 (bench kernel times + ncu counters)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out/carve; mkdir -p $O
B="--per-config '' --no-e2e --no-cpu-baseline --no-library"
km() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['roofline']['kernel_ms'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))" $1 2>&1; }
for rep in 1 2; do
  for c in 3 5; do
    if [ $c = 3 ]; then L="none 66 100"; else L="none 40 100"; fi
    for cv in $L; do
      f=$O/c${c}_cv${cv}_r$rep.json
      if [ $cv = none ]; then eval timeout 300 python bench.py --config $c $B > $f 2>/dev/null
      else eval HPDINV_SMEM_CARVEOUT=$cv timeout 300 python bench.py --config $c $B > $f 2>/dev/null; fi
      km $f >> $O/times.txt
    done
  done
  for g in 32 64; do
    f=$O/c5_l2f${g}_r$rep.json
    eval timeout 300 python tools/l2fetch_run.py $g --config 5 $B > $f 2>>$O/l2f.err
    km $f >> $O/times.txt
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__shared_mem_config_size,launch__occupancy_limit_shared_mem,l1tex__t_sector_hit_rate.pct
P="--per-config '' --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
for c in 3 5; do
  if [ $c = 3 ]; then L="none 66 100"; else L="none 40 100"; fi
  for cv in $L; do
    if [ $cv = none ]; then E=""; else E="HPDINV_SMEM_CARVEOUT=$cv"; fi
    eval $E timeout 300 ncu --metrics $M --clock-control none -k regex:k_grp -s 2 -c 1 --csv python bench.py --config $c $P > $O/ncu_c${c}_cv$cv.csv 2>/dev/null
  done
done
for g in 32 64; do
  eval timeout 300 ncu --metrics $M --clock-control none -k regex:k_grp -s 2 -c 1 --csv python tools/l2fetch_run.py $g --config 5 $P > $O/ncu_c5_l2f$g.csv 2>/dev/null
done
echo done >> $O/times.txt
