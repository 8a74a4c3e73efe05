# round 2 re-entry check: smoke, all GPU tests (no -x), config-4 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2c_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=30 > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2c_bench_c4.json 2> gpurun_out/r2c_bench_c4.err
for w in config2 config3; do timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench_$w.json 2> gpurun_out/r2c_bench_$w.err; done
echo done
