# round-2 iteration call: k_dmma parity + exact families + cfg4 bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact_api.py -x -q -p no:cacheprovider -k "64 or config_parity" > gpurun_out/t_dmma.log 2>&1; echo "pytest rc=$?" > gpurun_out/status2.txt
timeout 300 python bench.py --config 4 --per-config "" --no-e2e --no-library --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?" >> gpurun_out/status2.txt
