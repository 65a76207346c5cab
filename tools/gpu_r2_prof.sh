# ncu --set full of one workload's kernel, report kept in gpurun_out/.  Env: CFG, BATCH, KREGEX, TAG
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out
CMD="python bench.py --config ${CFG:-4} ${BATCH:+--batch $BATCH} --per-config '' --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
eval timeout 900 $CMD > $O/plain_${TAG:-x}.json 2>&1 && \
eval timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_}" -s 2 -c 1 -o $O/prof_${TAG:-x} $CMD > $O/ncu_${TAG:-x}.log 2>&1
echo "rc=$?" > $O/status_prof_${TAG:-x}.txt
