# k_grp staged-I/O check: GPU tests, then A/B (staged default vs HPDINV_GRP_NO_STAGE) on cfg3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_stage.log 2>&1; echo "pytest rc=$?" > $O/stage_status.txt
for v in base nostage base nostage; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_1111_4144_b200/libhpdinv_$v.so; fi
  HPDINV_LIB=$L timeout 300 python bench.py --config ${CFG:-3} --per-config '' --no-e2e --no-cpu-baseline --no-library --steps 20 --warmup 3 >> $O/ab_stage_$v.json 2>> $O/ab_stage_$v.err
done
echo done >> $O/stage_status.txt
