#!/bin/bash
# First-light GPU call: box facts, FP peaks, smoke, GPU tests, bench, ncu launch list + one
# full capture of the top kernel.  Usage (under gpurun): bash tools/gpu_check.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
{ nvidia-smi; nproc; lscpu | grep -E "Model name|^CPU\(s\)"; } > $O/box.txt 2>&1
./tools/peaks > $O/peaks.json 2>&1
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "${PYTEST_K:-not full_size}" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > $O/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_reg|k_generic|k_lane|k_cta" --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reg|k_generic|k_lane|k_cta" -s 5 -c 1 -o $O/prof_cfg2 $CMD > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/status.txt
