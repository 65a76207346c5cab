# A/B of library variants on one workload, interleaved twice.  Env: CFG, VARIANTS (besides base), TESTS=1 runs the GPU tests first
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_ab.log 2>&1; echo "pytest rc=$?" > $O/ab_status.txt; fi
for r in 1 2; do for v in base $VARIANTS; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_1111_4144_b200/libhpdinv_$v.so; fi
  HPDINV_LIB=$L timeout 300 python bench.py --config ${CFG:-3} --per-config '' --no-e2e --no-cpu-baseline --no-library --steps 20 --warmup 3 >> $O/ab_${v}_cfg${CFG:-3}.json 2>> $O/ab_${v}_cfg${CFG:-3}.err
done; done
echo done >> $O/ab_status.txt
