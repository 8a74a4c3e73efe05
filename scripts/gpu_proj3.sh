cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "tier2 or spans or degenerate or small_rrs or wrappers" > gpurun_out/proj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/proj_tests.log
timeout 600 python bench.py --workload config2 --steps 2 --warmup 1 --batch 256 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload config3 --steps 2 --warmup 1 --batch 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
