cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; O=gpurun_out
for c in 3 5; do
CMD="python bench.py --config $c --per-config '' --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-library"
eval timeout 600 $CMD > $O/plain_cfg$c.json 2>&1
eval timeout 900 ncu --set full -f --clock-control none --import-source on -k regex:"k_" -s 2 -c 1 -o $O/prof_cfg$c $CMD > $O/ncu_cfg$c.log 2>&1
echo "cfg$c rc=$?" >> $O/status35.txt
done
