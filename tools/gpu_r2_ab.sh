# A/B of library variants (HPDINV_LIB) on one workload.  Env: CFG, VARIANTS, STEPS
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out
for v in base $VARIANTS; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_1111_4144_b200/libhpdinv_$v.so; fi
  HPDINV_LIB=$L timeout 300 python bench.py --config ${CFG:-3} --per-config '' --no-e2e --no-cpu-baseline --no-library --steps ${STEPS:-20} --warmup 3 > $O/ab_${v}_cfg${CFG:-3}.json 2> $O/ab_${v}_cfg${CFG:-3}.err
done
